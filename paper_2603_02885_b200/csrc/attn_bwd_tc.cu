// attn_bwd_tc.cu — backward of the causal attention inside packed sequences
// (attn_tc.cu's forward) on tcgen05.
// With P = exp(scale S - lse), D = rowsum(dO o O) (mux_attn_bwd_pre_kernel):
//   dS = P o (dP - D),  dP = dO V^T,  dQ = scale dS K,  dK = scale dS^T Q,  dV = P^T dO.
// Two kernels, each output element owned by one CTA (no atomics: the result
// is bit-reproducible):
//
// dQ kernel — CTA = 128 query rows of one head (TMEM lanes = queries); key
//   tiles of 64, one K/V stage (112 KB smem, 256 TMEM columns: two CTAs per
//   SM hide each other's load and softmax latency).  Per tile: S = Q K^T and
//   dP = dO V^T (M=128, N=64, into TMEM), one thread per query row forms dS
//   (bf16, K-major smem), then dQ += dS K (M=128, N=128, K=64; K read MN-major).
//   TMEM: S 64 | dP 64 | dQ 128 columns.
// dV and dK kernels (one template, two launches) — CTA = 128 key rows of one
//   KV head (TMEM lanes = keys); query tiles of 64 of every q head of the
//   group through a TMA ring (2 stages for dV, 1 for dK).  Per tile: S^T = K Q^T (and, for dK,
//   dP^T = V dO^T) (M=128, N=64), one thread per key row forms P^T (dV) or
//   dS^T (dK) in bf16 (K-major smem), then dV += P^T dO or dK += dS^T Q
//   (M=128, N=128, K=64; dO, Q read MN-major).  Splitting dV from dK costs
//   one extra S^T product but keeps each CTA at 256 TMEM columns and <= 112 KB
//   of smem, so two CTAs share an SM.
// Warps 0-3: softmax-gradient + epilogue (TMEM lane quadrants), warp 4: MMA
// issuer, warp 5: TMA producer and TMEM allocator.
#include <climits>
#include <cmath>

#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

namespace {
constexpr uint32_t kSub128 = 128 * 128;  // [128 rows x 128 B] swizzled subtile (16 KB)
constexpr uint32_t kSub64 = 64 * 128;    // [64 rows x 128 B] (8 KB)
constexpr int kThreadsB = 192;
constexpr float kLog2eB = 1.4426950408889634f;

__device__ __forceinline__ uint64_t kdesc(uint32_t base, uint32_t sub, int k) {
  // K-major operand: subtiles of 64 elements (128 B rows) `sub` bytes apart; k-step k = 16 elements
  return make_desc(desc_lo(base + (k >> 2) * sub + (k & 3) * 32, 16), desc_hi(1024));
}
__device__ __forceinline__ uint64_t mdesc(uint32_t base, uint32_t atom, int k) {
  // MN-major operand: atoms of 64 N-elements (128 B) x rows, `atom` bytes apart; k-step = 16 rows
  return make_desc(desc_lo(base + k * 16 * 128, atom), desc_hi(1024));
}
// one thread's 64-element bf16 row -> swizzled K-major row (128 B) of a tile
__device__ __forceinline__ void store_row64(uint8_t* tile, int row, const uint32_t (&w)[32]) {
  uint8_t* prow = tile + row * 128;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    *reinterpret_cast<uint4*>(prow + ((q ^ (row & 7)) << 4)) = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2],
                                                                          w[4 * q + 3]);
}
}  // namespace

// =========================================================================== D
// D[r, h] = sum_d dO[r, h, d] O[r, h, d]: 16 threads per (row, head), 16-byte loads,
// whole warps iterate together (a half-warp past the end contributes nothing),
// half-warp shuffle reduction (grid-stride over rows x heads).
__global__ void __launch_bounds__(256) mux_attn_bwd_pre_kernel(int R, int H, const __nv_bfloat16* dO,
                                                              long long lddo, const __nv_bfloat16* O,
                                                              long long ldo, float* D) {
  griddep_wait();
  griddep_launch_dependents();
  const long long total = static_cast<long long>(R) * H * 16;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i - (threadIdx.x & 31) < total;
       i += stride) {
    const bool live = i < total;
    const long long rh = i >> 4;
    const int c = static_cast<int>(i & 15);
    float acc = 0.f;
    if (live) {
      const long long r = rh / H;
      const int h = static_cast<int>(rh - r * H);
      const uint4 a = *reinterpret_cast<const uint4*>(dO + r * lddo + h * 128 + c * 8);
      const uint4 b = *reinterpret_cast<const uint4*>(O + r * ldo + h * 128 + c * 8);
      const uint32_t x[4] = {a.x, a.y, a.z, a.w}, y[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        acc += __uint_as_float(x[e] << 16) * __uint_as_float(y[e] << 16) +
               __uint_as_float(x[e] & 0xFFFF0000u) * __uint_as_float(y[e] & 0xFFFF0000u);
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (live && c == 0) D[rh] = acc;
  }
}

// =========================================================================== dQ
// smem: Q 32 KB | dO 32 KB | dS 16 KB | K 16 KB, V 16 KB  (112 KB) | barriers
#ifndef MUX_DQ_STAGES
#define MUX_DQ_STAGES 1   // A/B builds: 2 (then 144 KB of smem, one CTA per SM)
#endif
constexpr int kDqStages = MUX_DQ_STAGES;
__global__ void __launch_bounds__(kThreadsB, kDqStages == 1 ? 2 : 1)
    mux_attn_dq_tc_kernel(const __grid_constant__ AttnBwdTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  constexpr uint32_t oQ = 0, oDO = 2 * kSub128, oDS = 4 * kSub128, oKV = 5 * kSub128;
  constexpr uint32_t kStage = 4 * kSub64;  // K 16 KB + V 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + oKV + kDqStages * kStage);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* sd_full = bars + 5;   // S and dP in TMEM
  uint64_t* ds_full = bars + 6;   // dS in smem (4 warp arrivals)
  uint64_t* dq_done = bars + 7;   // dQ += dS K complete
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 8);
  int* s_lohi = reinterpret_cast<int*>(bars + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * 128;
  const int h = blockIdx.y;
  const int hk = h / (p.H / p.Hkv);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(sd_full, 1);
    mbar_init(ds_full, 4);
    mbar_init(dq_done, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc<256>(tmem_holder);
  griddep_wait();
  griddep_launch_dependents();
  if (warp == 0) {
    int lo = INT_MAX, hi = -1;
    for (int i = lane; i < 128; i += 32) {
      const int r = q0 + i;
      if (r < p.R) {
        const int rs = p.row_start[r];
        if (rs >= 0) {
          lo = min(lo, rs);
          hi = max(hi, r);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      s_lohi[0] = lo;
      s_lohi[1] = hi;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int lo = s_lohi[0], hi = s_lohi[1];
  const int ntiles = hi >= 0 ? (hi - lo) / 64 + 1 : 0;
  const uint32_t sb = smem_u32(smem);
  if (warp == 5) {
    if (ntiles > 0 && elect_one_sync()) {
      mbar_arrive_expect_tx(q_full, 4 * kSub128);
      for (int s2 = 0; s2 < 2; ++s2) {
        tma_load_2d(&p.map_q128, q_full, smem + oQ + s2 * kSub128, h * 128 + 64 * s2, q0);
        tma_load_2d(&p.map_do128, q_full, smem + oDO + s2 * kSub128, h * 128 + 64 * s2, q0);
      }
      for (int j = 0; j < ntiles; ++j) {
        const int s = j % kDqStages;
        mbar_wait(&kv_empty[s], ((j / kDqStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[s], kStage);
        uint8_t* st = smem + oKV + s * kStage;
        const int kt = lo + 64 * j;
        for (int s2 = 0; s2 < 2; ++s2) {
          tma_load_2d(&p.map_k64, &kv_full[s], st + s2 * kSub64, hk * 128 + 64 * s2, kt);
          tma_load_2d(&p.map_v64, &kv_full[s], st + 2 * kSub64 + s2 * kSub64, hk * 128 + 64 * s2, kt);
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    if (ntiles > 0) {
      constexpr uint32_t kId64 = idesc_bf16(128, 64, false, false);   // S, dP: both K-major
      constexpr uint32_t kId128 = idesc_bf16(128, 128, false, true);  // dS K: K read MN-major
      const uint32_t tS = tmem, tP = tmem + 64, tQ = tmem + 128;
      mbar_wait(q_full, 0);
      tc_fence_after();
      // per step: first the dQ product of tile j-1 (it frees tile j-1's K/V stage, which
      // a single-stage ring needs before tile j can land), then S, dP of tile j
      for (int j = 0; j <= ntiles; ++j) {
        if (j > 0) {
          const int jp = j - 1;
          mbar_wait(ds_full, jp & 1);  // dS_{j-1} written, S/dP of tile j-1 read
          tc_fence_after();
          const uint32_t st = sb + oKV + (jp % kDqStages) * kStage;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16(tQ, kdesc(sb + oDS, kSub128, k), mdesc(st, kSub64, k), kId128, (jp > 0 || k > 0) ? 1u : 0u);
            mma_commit(dq_done);
            mma_commit(&kv_empty[jp % kDqStages]);
          }
          __syncwarp();
        }
        if (j < ntiles) {
          mbar_wait(&kv_full[j % kDqStages], (j / kDqStages) & 1);
          tc_fence_after();
          const uint32_t st = sb + oKV + (j % kDqStages) * kStage;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              mma_bf16(tS, kdesc(sb + oQ, kSub128, k), kdesc(st, kSub64, k), kId64, k > 0 ? 1u : 0u);
              mma_bf16(tP, kdesc(sb + oDO, kSub128, k), kdesc(st + 2 * kSub64, kSub64, k), kId64, k > 0 ? 1u : 0u);
            }
            mma_commit(sd_full);
          }
          __syncwarp();
        }
      }
    }
  } else {
    const int row = warp * 32 + lane;
    const int r = q0 + row;
    const int rlo = r < p.R ? p.row_start[r] : -1;
    const float l2 = rlo >= 0 ? p.lse[static_cast<long long>(r) * p.H + h] * kLog2eB : 0.f;
    const float Dr = rlo >= 0 ? p.D[static_cast<long long>(r) * p.H + h] : 0.f;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t tS = tmem + lane_off, tP = tS + 64, tQ = tS + 128;
    for (int j = 0; j < ntiles; ++j) {
      const int kt = lo + 64 * j;
      mbar_wait(sd_full, j & 1);
      tc_fence_after();
      uint32_t sv[2][32], pv[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tmem_ld32(tS + 32 * c, sv[c]);
        tmem_ld32(tP + 32 * c, pv[c]);
      }
      tmem_ld_wait();
      uint32_t w[32];
      // interior tile (no key of it masked for any row of the warp): no per-element mask
      if (__all_sync(0xffffffffu, rlo >= 0 && kt >= rlo && kt + 63 <= r)) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float d2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float pr = ex2_approx(fmaf(__uint_as_float(sv[c][2 * i + e]), p.scale_log2, -l2));
              d2[e] = pr * (__uint_as_float(pv[c][2 * i + e]) - Dr);
            }
            w[16 * c + i] = pack_bf16x2(d2[0], d2[1]);
          }
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float d2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int key = kt + 32 * c + 2 * i + e;
              const bool ok = rlo >= 0 && key >= rlo && key <= r;
              const float pr = ok ? ex2_approx(fmaf(__uint_as_float(sv[c][2 * i + e]), p.scale_log2, -l2)) : 0.f;
              d2[e] = pr * (__uint_as_float(pv[c][2 * i + e]) - Dr);
            }
            w[16 * c + i] = pack_bf16x2(d2[0], d2[1]);
          }
      }
      if (j > 0) {  // dQ += dS_{j-1} K_{j-1} must have read the dS buffer
        mbar_wait(dq_done, (j - 1) & 1);
        tc_fence_after();
      }
      store_row64(smem + oDS, row, w);
      fence_async_shared();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
    }
    if (r < p.R) {
      uint4* dst = reinterpret_cast<uint4*>(p.dq + static_cast<long long>(r) * p.lddq + h * 128);
      if (ntiles > 0) {
        mbar_wait(dq_done, (ntiles - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld32(tQ + 32 * c, v);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float s = p.scale;
            dst[4 * c + q] = make_uint4(
                pack_bf16x2(__uint_as_float(v[8 * q]) * s, __uint_as_float(v[8 * q + 1]) * s),
                pack_bf16x2(__uint_as_float(v[8 * q + 2]) * s, __uint_as_float(v[8 * q + 3]) * s),
                pack_bf16x2(__uint_as_float(v[8 * q + 4]) * s, __uint_as_float(v[8 * q + 5]) * s),
                pack_bf16x2(__uint_as_float(v[8 * q + 6]) * s, __uint_as_float(v[8 * q + 7]) * s));
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) dst[c] = make_uint4(0, 0, 0, 0);
      }
    } else if (ntiles > 0) {
      mbar_wait(dq_done, (ntiles - 1) & 1);  // keep TMEM alive until the last MMA is done
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// =========================================================================== dK, dV
// smem: K 32 KB | [dK: V 32 KB] | P^T or dS^T 16 KB | Q 16 KB, dO 16 KB (one stage) | scalars | barriers
// Q/dO ring depth: dV (no V tile) fits two stages in 112 KB, dK one; either way two CTAs share an SM
#ifndef MUX_DK_STAGES
#define MUX_DK_STAGES 1   // A/B builds: 2 (then 144 KB of smem for dK, one CTA per SM)
#endif
template <bool kDK>
constexpr int qd_stages() { return kDK ? MUX_DK_STAGES : 2; }
template <bool kDK>
__global__ void __launch_bounds__(kThreadsB, (kDK && MUX_DK_STAGES > 1) ? 1 : 2)
    mux_attn_dkdv_tc_kernel(const __grid_constant__ AttnBwdTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  constexpr uint32_t oK = 0, oV = 2 * kSub128, oT = (kDK ? 4 : 2) * kSub128, oQD = oT + kSub128;
  constexpr uint32_t kStage = 4 * kSub64;  // Q 16 KB + dO 16 KB
  constexpr int kNS = qd_stages<kDK>();
  float* sc = reinterpret_cast<float*>(smem + oQD + kNS * kStage);  // [3][64]: lse2, D, row_start
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + oQD + kNS * kStage + 3 * 64 * 4);
  uint64_t* kv_full = bars + 0;
  uint64_t* qd_full = bars + 1;   // [2]
  uint64_t* qd_empty = bars + 3;  // [2]
  uint64_t* sd_full = bars + 5;
  uint64_t* pd_full = bars + 6;   // P^T and dS^T in smem (4 warp arrivals)
  uint64_t* mm_done = bars + 7;   // dV, dK MMAs of the tile complete
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 8);
  int* s_i = reinterpret_cast<int*>(bars + 9);  // first, last, qend
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = blockIdx.x * 128;
  const int hk = blockIdx.y;
  const int G = p.H / p.Hkv;
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qd_full[s], 1);
      mbar_init(&qd_empty[s], 1);
    }
    mbar_init(sd_full, 1);
    mbar_init(pd_full, 4);
    mbar_init(mm_done, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc<256>(tmem_holder);
  griddep_wait();
  griddep_launch_dependents();
  if (warp == 0) {  // valid keys of the tile and the end of the last one's sequence
    int first = INT_MAX, last = -1;
    for (int i = lane; i < 128; i += 32) {
      const int r = k0 + i;
      if (r < p.R && p.row_start[r] >= 0) {
        first = min(first, r);
        last = max(last, r);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
      last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    }
    int qend = last;
    if (last >= 0) {
      const int s = p.row_start[last];
      for (int base = last + 1; base < p.R; base += 32) {
        const int r = base + lane;
        const bool same = r < p.R && p.row_start[r] == s;
        const unsigned m = __ballot_sync(0xffffffffu, same);
        if (m != 0xffffffffu) {
          qend = base + __ffs(~m) - 2;
          break;
        }
        qend = base + 31;
      }
      qend = min(qend, p.R - 1);
    }
    if (lane == 0) {
      s_i[0] = first;
      s_i[1] = last;
      s_i[2] = qend;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int first = s_i[0], last = s_i[1], qend = s_i[2];
  const int nq = last >= 0 ? (qend - first) / 64 + 1 : 0;  // query tiles per head
  const int steps = nq * G;
  const uint32_t sb = smem_u32(smem);
  if (warp == 5) {
    if (steps > 0) {
      if (elect_one_sync()) {
        mbar_arrive_expect_tx(kv_full, (kDK ? 4 : 2) * kSub128);
        for (int s2 = 0; s2 < 2; ++s2) {
          tma_load_2d(&p.map_k128, kv_full, smem + oK + s2 * kSub128, hk * 128 + 64 * s2, k0);
          if (kDK) tma_load_2d(&p.map_v128, kv_full, smem + oV + s2 * kSub128, hk * 128 + 64 * s2, k0);
        }
      }
      __syncwarp();
      for (int j = 0; j < steps; ++j) {
        const int s = j % kNS;
        const int hh = j / nq, qi = j - hh * nq;
        const int h = hk * G + hh;
        const int qt = first + 64 * qi;
        mbar_wait(&qd_empty[s], ((j / kNS) & 1) ^ 1);
        if (elect_one_sync()) {
          mbar_arrive_expect_tx(&qd_full[s], kStage);
          uint8_t* st = smem + oQD + s * kStage;
          for (int s2 = 0; s2 < 2; ++s2) {
            tma_load_2d(&p.map_q64, &qd_full[s], st + s2 * kSub64, h * 128 + 64 * s2, qt);
            tma_load_2d(&p.map_do64, &qd_full[s], st + 2 * kSub64 + s2 * kSub64, h * 128 + 64 * s2, qt);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 4) {
    if (steps > 0) {
      constexpr uint32_t kId64 = idesc_bf16(128, 64, false, false);   // S^T, dP^T: K-major
      constexpr uint32_t kId128 = idesc_bf16(128, 128, false, true);  // dV, dK: dO / Q read MN-major
      const uint32_t tS = tmem, tP = tmem + 64, tAcc = tmem + 128;
      mbar_wait(kv_full, 0);
      tc_fence_after();
      // per step: first the accumulate of step j-1 (frees its Q/dO stage), then S^T (, dP^T) of step j
      for (int j = 0; j <= steps; ++j) {
        if (j > 0) {
          const int jp = j - 1;
          mbar_wait(pd_full, jp & 1);
          tc_fence_after();
          const uint32_t st = sb + oQD + (jp % kNS) * kStage;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)  // dV += P^T dO  or  dK += dS^T Q
              mma_bf16(tAcc, kdesc(sb + oT, kSub128, k), mdesc(st + (kDK ? 0 : 2 * kSub64), kSub64, k), kId128,
                       (jp > 0 || k > 0) ? 1u : 0u);
            mma_commit(mm_done);
            mma_commit(&qd_empty[jp % kNS]);
          }
          __syncwarp();
        }
        if (j < steps) {
          mbar_wait(&qd_full[j % kNS], (j / kNS) & 1);
          tc_fence_after();
          const uint32_t st = sb + oQD + (j % kNS) * kStage;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              mma_bf16(tS, kdesc(sb + oK, kSub128, k), kdesc(st, kSub64, k), kId64, k > 0 ? 1u : 0u);
              if (kDK)
                mma_bf16(tP, kdesc(sb + oV, kSub128, k), kdesc(st + 2 * kSub64, kSub64, k), kId64,
                         k > 0 ? 1u : 0u);
            }
            mma_commit(sd_full);
          }
          __syncwarp();
        }
      }
    }
  } else {
    const int row = warp * 32 + lane;
    const int kr = k0 + row;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t tS = tmem + lane_off, tP = tS + 64, tAcc = tS + 128;
    for (int j = 0; j < steps; ++j) {
      const int qi = j % nq;
      const int qt = first + 64 * qi;
      float* scs = sc;
      const int* rss = reinterpret_cast<const int*>(scs) + 128;
      {
        asm volatile("bar.sync 1, 128;" ::: "memory");  // everyone is done with the previous step's scalars
        const int hh = j / nq;
        const int h = hk * G + hh;
        if (row < 64) {
          const int r = qt + row;
          const int rs = r < p.R ? p.row_start[r] : -1;
          scs[row] = rs >= 0 ? p.lse[static_cast<long long>(r) * p.H + h] * kLog2eB : 0.f;
          reinterpret_cast<int*>(scs)[128 + row] = rs;
        } else if (kDK) {
          const int r = qt + row - 64;
          scs[row] = r < p.R ? p.D[static_cast<long long>(r) * p.H + h] : 0.f;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 softmax warps
      }
      mbar_wait(sd_full, j & 1);
      tc_fence_after();
      uint32_t sv[2][32], pv[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tmem_ld32(tS + 32 * c, sv[c]);
        if (kDK) tmem_ld32(tP + 32 * c, pv[c]);
      }
      tmem_ld_wait();
      uint32_t w[32];  // P^T (dV) or dS^T = P^T o (dP^T - D) (dK), bf16 pairs
      // interior tile: every query of the tile sees every key row of the warp
      // (kr <= qt, kr >= max row_start, no invalid query): no per-element mask
      int rs_max = max(rss[lane], rss[32 + lane]);
      int rs_min = min(rss[lane], rss[32 + lane]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rs_max = max(rs_max, __shfl_xor_sync(0xffffffffu, rs_max, o));
        rs_min = min(rs_min, __shfl_xor_sync(0xffffffffu, rs_min, o));
      }
      if (__all_sync(0xffffffffu, rs_min >= 0 && kr >= rs_max && kr <= qt)) {
        const float4* lse4 = reinterpret_cast<const float4*>(scs);
        const float4* d4 = reinterpret_cast<const float4*>(scs + 64);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float4 l4 = lse4[(32 * c + 2 * i) >> 2];
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
            float dv[4] = {0.f, 0.f, 0.f, 0.f};
            if (kDK) {
              const float4 t = d4[(32 * c + 2 * i) >> 2];
              dv[0] = t.x; dv[1] = t.y; dv[2] = t.z; dv[3] = t.w;
            }
            float x[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float pr = ex2_approx(fmaf(__uint_as_float(sv[c][2 * i + e]), p.scale_log2, -lv[e]));
              x[e] = kDK ? pr * (__uint_as_float(pv[c][2 * i + e]) - dv[e]) : pr;
            }
            w[16 * c + i] = pack_bf16x2(x[0], x[1]);
            w[16 * c + i + 1] = pack_bf16x2(x[2], x[3]);
          }
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = 32 * c + 2 * i + e;
              const int qr = qt + col;
              const int rs = rss[col];
              const bool ok = rs >= 0 && rs <= kr && kr <= qr;
              const float pr =
                  ok ? ex2_approx(fmaf(__uint_as_float(sv[c][2 * i + e]), p.scale_log2, -scs[col])) : 0.f;
              x[e] = kDK ? pr * (__uint_as_float(pv[c][2 * i + e]) - scs[64 + col]) : pr;
            }
            w[16 * c + i] = pack_bf16x2(x[0], x[1]);
          }
      }
      if (j > 0) {  // the previous tile's accumulate MMA must have read the P^T / dS^T tile
        mbar_wait(mm_done, (j - 1) & 1);
        tc_fence_after();
      }
      store_row64(smem + oT, row, w);
      fence_async_shared();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(pd_full);
    }
    if (kr < p.R) {
      uint4* dst = kDK ? reinterpret_cast<uint4*>(p.dk + static_cast<long long>(kr) * p.lddk + hk * 128)
                       : reinterpret_cast<uint4*>(p.dv + static_cast<long long>(kr) * p.lddv + hk * 128);
      if (steps > 0) {
        mbar_wait(mm_done, (steps - 1) & 1);
        tc_fence_after();
        const float s = kDK ? p.scale : 1.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld32(tAcc + 32 * c, v);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[4 * c + q] = make_uint4(
                pack_bf16x2(__uint_as_float(v[8 * q]) * s, __uint_as_float(v[8 * q + 1]) * s),
                pack_bf16x2(__uint_as_float(v[8 * q + 2]) * s, __uint_as_float(v[8 * q + 3]) * s),
                pack_bf16x2(__uint_as_float(v[8 * q + 4]) * s, __uint_as_float(v[8 * q + 5]) * s),
                pack_bf16x2(__uint_as_float(v[8 * q + 6]) * s, __uint_as_float(v[8 * q + 7]) * s));
        }
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) dst[c] = make_uint4(0, 0, 0, 0);
      }
    } else if (steps > 0) {
      mbar_wait(mm_done, (steps - 1) & 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

constexpr size_t kDqSmemTc = 5 * kSub128 + kDqStages * 4 * kSub64 + 256;
template <bool kDK>
constexpr size_t dkdv_smem() {
  return ((kDK ? 4 : 2) + 1) * kSub128 + qd_stages<kDK>() * 4 * kSub64 + 3 * 64 * 4 + 256;  // 115712 B = half an SM
}

cudaError_t launch_attn_bwd_pre(int R, int H, const void* dO, long long lddo, const void* o, long long ldo,
                                float* D, cudaStream_t s) {
  const long long threads = static_cast<long long>(R) * H * 16;
  if (threads == 0) return cudaSuccess;
  long long blocks = (threads + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_pdl(mux_attn_bwd_pre_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, R, H,
                    static_cast<const __nv_bfloat16*>(dO), lddo, static_cast<const __nv_bfloat16*>(o), ldo, D);
}

template <bool kDK>
cudaError_t configure_dkdv() {
  cudaError_t e = cudaFuncSetAttribute(mux_attn_dkdv_tc_kernel<kDK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(dkdv_smem<kDK>()));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(mux_attn_dkdv_tc_kernel<kDK>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  return e;
}

cudaError_t launch_attn_bwd_tc(const AttnBwdTcParams& p, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t ce = once_per_device(configured, [] {
    cudaError_t e = cudaFuncSetAttribute(mux_attn_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kDqSmemTc));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mux_attn_dq_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess) e = configure_dkdv<false>();
    if (e == cudaSuccess) e = configure_dkdv<true>();
    return e;
  });
  if (ce != cudaSuccess) return ce;
  if (p.R == 0) return cudaSuccess;
  const dim3 gk((p.R + 127) / 128, p.Hkv);
  cudaError_t e = launch_pdl(mux_attn_dkdv_tc_kernel<false>, gk, dim3(kThreadsB), dkdv_smem<false>(), s, p);
  if (e == cudaSuccess) e = launch_pdl(mux_attn_dkdv_tc_kernel<true>, gk, dim3(kThreadsB), dkdv_smem<true>(), s, p);
  if (e != cudaSuccess) return e;
  return launch_pdl(mux_attn_dq_tc_kernel, dim3((p.R + 127) / 128, p.H), dim3(kThreadsB), kDqSmemTc, s, p);
}

}  // namespace mux
