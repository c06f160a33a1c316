// attn_tc.cu — forward of the causal attention inside packed sequences
// (same operation as attn.cu) on the 5th-gen
// tensor cores: tcgen05.mma with both products accumulated in TMEM.
//
// One CTA = 128 query rows (= the 128 TMEM lanes) of one head; key tiles of
// 64 rows stream through a 2-stage TMA ring (112 KB of smem and 256 TMEM
// columns per CTA: two CTAs share an SM, so one's prologue, softmax and
// epilogue overlap the other's MMAs).  Per key tile j:
//   S_j = Q K_j^T           tcgen05.mma M=128 N=64, A = Q (K-major smem),
//                           B = K_j (K-major smem)          -> TMEM cols [64 (j&1), +64)
//   softmax (one thread per query row, tcgen05.ld of its S row): mask to
//   [row_start, row], running max with lazy rescaling (the O accumulator is
//   rescaled in TMEM only when the max grows by more than 2^8), P_j = exp2(.)
//   as bf16 into a 128 B-swizzled K-major smem tile
//   O += P_j V_j            tcgen05.mma M=128 N=128 K=64, A = P_j (smem),
//                           B = V_j (MN-major smem)         -> TMEM cols [128,256)
// S is double-buffered in TMEM: S_{j+1} is computed while softmax j runs (it
// only needs softmax j-1 to have read its buffer), so the tensor core and the
// softmax overlap instead of alternating.
// Warps 0-3: softmax + epilogue (TMEM lane quadrants), warp 4: MMA issuer,
// warp 5: TMA producer and TMEM allocator.
#include <climits>
#include <cmath>

#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {


namespace {
constexpr int kT = 128;                       // query rows per CTA (TMEM lanes)
constexpr int kTN = 64;                       // keys per tile
constexpr uint32_t kSubQ = 128 * 128;         // Q: [128 rows x 128 B] swizzled subtile (16 KB), 2 per tile
constexpr uint32_t kSubK = 64 * 128;          // K, V: [64 rows x 128 B] subtile (8 KB), 2 per tile
constexpr uint32_t kTileQ = 2 * kSubQ, kTileK = 2 * kSubK;
// Q 32 KB | P [128 q x 64 keys] 16 KB | KV stage s: K (16 KB), V (16 KB) | barriers
constexpr uint32_t kSmemQ = 0, kSmemP = kTileQ, kSmemKV = kTileQ + kSubQ;
constexpr uint32_t kSmemData = kSmemKV + 2 * 2 * kTileK;   // 112 KB
constexpr uint32_t kSmemBytes = kSmemData + 256;           // dynamic smem base is 1024-aligned (no static smem)
constexpr int kThreads = 192;
constexpr float kLazy = 8.f;                  // rescale O only when the max grows by > 2^8

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
}  // namespace

__global__ void __launch_bounds__(kThreads, 2) mux_attn_fwd_tc_kernel(const __grid_constant__ AttnTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1 KB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemData);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;   // [2] S buffer b holds S_j (j & 1 == b)
  uint64_t* s_free = bars + 7;   // [2] the 4 softmax warps have read S buffer b
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 11);
  int* s_lohi = reinterpret_cast<int*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * kT;
  const int h = blockIdx.y;
  const int hk = h / (p.H / p.Hkv);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 5) {
    if (lane == 0) {
      tma_prefetch(&p.map_q);
      tma_prefetch(&p.map_k);
      tma_prefetch(&p.map_v);
    }
    tmem_alloc<256>(tmem_holder);
  }
  griddep_wait();
  griddep_launch_dependents();
  // key range of the tile: [min row_start over valid rows, last valid row]
  if (warp == 0) {
    int lo = INT_MAX, hi = -1;
    for (int i = lane; i < kT; i += 32) {
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
  const int ntiles = hi >= 0 ? (hi - lo) / kTN + 1 : 0;
  const uint32_t sbase = smem_u32(smem);

  if (warp == 5) {
    // =========================== TMA producer
    if (ntiles > 0 && elect_one_sync()) {
      mbar_arrive_expect_tx(q_full, kTileQ);
      for (int s2 = 0; s2 < 2; ++s2)
        tma_load_2d(&p.map_q, q_full, smem + kSmemQ + s2 * kSubQ, h * 128 + 64 * s2, q0);
      for (int j = 0; j < ntiles; ++j) {
        const int s = j & 1;
        mbar_wait(&kv_empty[s], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[s], 2 * kTileK);
        uint8_t* sk = smem + kSmemKV + s * 2 * kTileK;
        const int kt = lo + j * kTN;
        for (int s2 = 0; s2 < 2; ++s2) {
          tma_load_2d(&p.map_k, &kv_full[s], sk + s2 * kSubK, hk * 128 + 64 * s2, kt);
          tma_load_2d(&p.map_v, &kv_full[s], sk + kTileK + s2 * kSubK, hk * 128 + 64 * s2, kt);
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    // =========================== MMA issuer
    if (ntiles > 0) {
      constexpr uint32_t kIdS = idesc_bf16(128, kTN, false, false);  // Q K^T: both K-major
      constexpr uint32_t kIdO = idesc_bf16(128, 128, false, true);   // P V: V is MN-major (d contiguous)
      constexpr uint32_t kHi = desc_hi(1024);
      const uint32_t tO = tmem + 128;  // S_j in TMEM columns [64 (j & 1), +64)
      // K-major operand = subtiles of 64 elems (128 B rows) `sub` bytes apart; k-step k (16 elems)
      auto kmaj = [&](uint32_t base, uint32_t sub, int k) {
        return make_desc(desc_lo(base + (k >> 2) * sub + (k & 3) * 32, 16), kHi);
      };
      // V [64 keys x 128 d], MN-major: 2 atoms of 64 d (LBO = 8 KB), k-step = 16 key rows
      auto vmaj = [&](uint32_t base, int k) { return make_desc(desc_lo(base + k * 16 * 128, kSubK), kHi); };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= ntiles; ++j) {
        if (j < ntiles) {
          mbar_wait(&kv_full[j & 1], (j >> 1) & 1);
          if (j >= 2) mbar_wait(&s_free[j & 1], ((j >> 1) - 1) & 1);  // softmax j-2 read this buffer
          tc_fence_after();
          const uint32_t sk = sbase + kSmemKV + (j & 1) * 2 * kTileK;
          const uint32_t tS = tmem + 64u * static_cast<uint32_t>(j & 1);
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              mma_bf16(tS, kmaj(sbase + kSmemQ, kSubQ, k), kmaj(sk, kSubK, k), kIdS, k > 0 ? 1u : 0u);
            mma_commit(&s_full[j & 1]);
          }
          __syncwarp();
        } else {
          mbar_wait(p_full, (j - 1) & 1);
          tc_fence_after();
        }
        if (j > 0) {
          const int jp = j - 1;
          if (j < ntiles) {  // softmax j-1 wrote P (the last iteration waited above)
            mbar_wait(p_full, jp & 1);
            tc_fence_after();
          }
          const uint32_t sv = sbase + kSmemKV + (jp & 1) * 2 * kTileK + kTileK;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < kTN / 16; ++k)
              mma_bf16(tO, kmaj(sbase + kSmemP, kSubQ, k), vmaj(sv, k), kIdO, (jp > 0 || k > 0) ? 1u : 0u);
            mma_commit(o_done);
            mma_commit(&kv_empty[jp & 1]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // =========================== softmax + epilogue (warps 0-3: TMEM lanes 32 w ..)
    const int row = warp * 32 + lane;
    const int r = q0 + row;
    const int rlo = r < p.R ? p.row_start[r] : -1;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t tO = tmem + lane_off + 128;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int kt = lo + j * kTN;
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[2][32];
      const uint32_t tS = tmem + lane_off + 64u * static_cast<uint32_t>(j & 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) tmem_ld32(tS + 32 * c, sv[c]);
      tmem_ld_wait();
      // S_j is in registers: its TMEM buffer may take S_{j+2} while this softmax runs
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[j & 1]);
      // Interior tiles (every key of the tile visible to every row of the warp) skip the
      // per-element mask: the kernel is instruction-bound, and the mask was most of it.
      const bool interior = __all_sync(0xffffffffu, rlo >= 0 && kt >= rlo && kt + kTN - 1 <= r);
      float mx = -INFINITY;
      if (interior) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(sv[c][i]));
        mx *= p.scale_log2;  // scale > 0: max commutes with the scaling
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int key = kt + 32 * c + i;
            const bool ok = rlo >= 0 && key >= rlo && key <= r;
            const float x = ok ? __uint_as_float(sv[c][i]) * p.scale_log2 : -INFINITY;
            sv[c][i] = __float_as_uint(x);
            mx = fmaxf(mx, x);
          }
      }
      // lazy rescaling: keep the running max unless it grew by more than kLazy (log2 units)
      float alpha = 1.f;
      const bool grow = mx > m_used + kLazy || (m_used == -INFINITY && mx > -INFINITY);
      if (grow) {
        alpha = m_used == -INFINITY ? 0.f : exp2f(m_used - mx);
        m_used = mx;
      }
      const float mu = m_used == -INFINITY ? 0.f : m_used;
      uint32_t pw[32];
      float sum = 0.f;
      // interior: sv holds raw scores, P = 2^(s * scale - mu) in one FFMA + one SFU op
      const float sc = interior ? p.scale_log2 : 1.f;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float a = ex2_approx(fmaf(__uint_as_float(sv[c][2 * i]), sc, -mu));
          const float b = ex2_approx(fmaf(__uint_as_float(sv[c][2 * i + 1]), sc, -mu));
          sum += a + b;
          pw[16 * c + i] = pack_bf16x2(a, b);
        }
      l = l * alpha + sum;
      // P_{j-1} V_{j-1} must be done before P is overwritten or O rescaled
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld32(tO + 32 * c, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st32(tO + 32 * c, ov);
          }
          tmem_st_wait();
        }
      }
      // P row (64 keys = one 128 B swizzled row of the K-major P tile)
      uint8_t* prow = smem + kSmemP + row * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(prow + ((q ^ (row & 7)) << 4)) =
            make_uint4(pw[4 * q], pw[4 * q + 1], pw[4 * q + 2], pw[4 * q + 3]);
      fence_async_shared();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 row, lse
    float ov_f[128];
    if (ntiles > 0) {
      mbar_wait(o_done, (ntiles - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        tmem_ld32(tO + 32 * c, ov);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) ov_f[32 * c + i] = __uint_as_float(ov[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 128; ++i) ov_f[i] = 0.f;
    }
    if (r < p.R) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(p.o + static_cast<long long>(r) * p.ldo + h * 128);
#pragma unroll
      for (int c = 0; c < 16; ++c)
        dst[c] = make_uint4(pack_bf16x2(ov_f[8 * c] * inv, ov_f[8 * c + 1] * inv),
                            pack_bf16x2(ov_f[8 * c + 2] * inv, ov_f[8 * c + 3] * inv),
                            pack_bf16x2(ov_f[8 * c + 4] * inv, ov_f[8 * c + 5] * inv),
                            pack_bf16x2(ov_f[8 * c + 6] * inv, ov_f[8 * c + 7] * inv));
      p.lse[static_cast<long long>(r) * p.H + h] = l > 0.f ? (m_used + log2f(l)) * 0.6931471805599453f : -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

cudaError_t launch_attn_fwd_tc(const AttnTcParams& p, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t ce = once_per_device(configured, [] {
    cudaError_t e = cudaFuncSetAttribute(mux_attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemBytes));
    if (e == cudaSuccess)  // the whole 228 KB as shared memory: two CTAs per SM
      e = cudaFuncSetAttribute(mux_attn_fwd_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return e;
  });
  if (ce != cudaSuccess) return ce;
  if (p.R == 0) return cudaSuccess;
  return launch_pdl(mux_attn_fwd_tc_kernel, dim3((p.R + kT - 1) / kT, p.H), dim3(kThreads), kSmemBytes, s, p);
}

}  // namespace mux
