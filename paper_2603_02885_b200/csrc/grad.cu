// grad.cu — segmented adapter-weight gradients on tcgen05 (sm_100a).
//
//   dA_t[j, k] = sum_{i in segments of t} Gs[i, j] X[i, k]     (fp32 [rank, K])
//   dB_t[n, j] = sum_{i in segments of t} dY[i, n] Hs[i, j]    (fp32 [N, rank])
//
// (Gs = s_t dY B_t and Hs = s_t X A_t^T carry the LoRA scale; chain rule of
// the north_star formula.)  Both are reductions over a task's
// tokens with a small output, HBM-bound (arithmetic intensity ~ rank FLOP/B):
// X and dY are each streamed from HBM exactly once.  A work unit is
// (task, 128 output rows of k or n); it runs a TMA -> smem -> tcgen05 pipeline
// over all 128-token blocks of the task's segments with M = 128 (k or n,
// MN-major A operand), N = 64 (rank padded, MN-major B operand), K = tokens.
// Token blocks never cross into another segment's rows: a block that extends
// past its segment end (segments are multiples of 64) only issues the MMAs of
// its valid 64 tokens.  Deterministic: one unit owns each output element and
// sums tokens in ascending order.  Ranks < 16 still use the tensor cores
// (zero-padded N = 64): the kernel is bound by streaming X/dY, not by MMA.
#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

constexpr uint32_t kGAtom = kGradBK * 128;            // 128 token rows x 128 B = 16 KB
constexpr uint32_t kGStageA = 2 * kGAtom;             // 128 output rows = 2 MN atoms
constexpr uint32_t kGPipeBytes = kGradStages * (kGStageA + kGAtom);  // 192 KB of stages
constexpr uint32_t kGradSmemBytes = kGPipeBytes + 1024 + 1024;
constexpr uint32_t kGradTmemCols = 512;               // 2 accumulators of up to 256 columns
constexpr uint32_t kGAccStride = 256;
constexpr int kGradThreads = 256;

__global__ void __launch_bounds__(kGradThreads, 1) mux_grad_kernel(const __grid_constant__ GradParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* pipe = smem;
  uint8_t* misc = smem + kGPipeBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(misc);
  uint64_t* empty_bar = full_bar + kGradStages;
  uint64_t* tfull_bar = empty_bar + kGradStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* so = reinterpret_cast<int*>(misc + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int stages = p.stages;
  const uint32_t stage_bytes = p.stage_bytes;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.map_x);
    tma_prefetch(&p.map_dy);
    tma_prefetch(&p.map_hs);
    tma_prefetch(&p.map_gs);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kGradTmemCols>(tmem_holder);
  griddep_wait();  // PDL: the prologue above overlaps the previous kernel
  griddep_launch_dependents();
  for (int i = threadIdx.x; i <= p.num_segs; i += blockDim.x) so[i] = p.seg_off[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int per_task = p.units_a + p.units_b;
  const int total_units = p.num_tasks * per_task;
  const int S = p.num_slices;
  // slice of dB unit `ub` (units of a task: dA first, then dB slice by slice)
  auto b_slice = [&](int ub) {
    int sc = 0;
    while (sc + 1 < S && ub >= p.b_units_off[sc + 1]) ++sc;
    return sc;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const int task = u / per_task;
        const int sub = u - task * per_task;
        const bool is_a = sub < p.units_a;
        // dA: rows k of X, all nb_a Gs boxes; dB: rows n of the slice's dY columns, its Hs box
        int col_a, col_b = 0, nb = 1;
        if (is_a) {
          col_a = sub * kGradBM;
          nb = p.nb_a;
        } else {
          const int ub = sub - p.units_a;
          const int sc = b_slice(ub);
          col_a = p.slice_off[sc] + (ub - p.b_units_off[sc]) * kGradBM;
          col_b = sc * p.r_cap;
        }
        const CUtensorMap* ma = is_a ? &p.map_x : &p.map_dy;
        const CUtensorMap* mb = is_a ? &p.map_gs : &p.map_hs;
        const uint32_t bytes = kGStageA + static_cast<uint32_t>(nb) * kGAtom;
        const uint64_t segs = p.task_segs[task];
        for (int s = 0; s < p.num_segs; ++s) {
          if (!((segs >> s) & 1ull)) continue;
          for (int tok = so[s]; tok < so[s + 1]; tok += kGradBK) {
            mbar_wait(&empty_bar[stage], phase ^ 1u);
            uint8_t* sa = pipe + stage * stage_bytes;
            mbar_arrive_expect_tx(&full_bar[stage], bytes);
            tma_load_2d(ma, &full_bar[stage], sa, col_a, tok);
            tma_load_2d(ma, &full_bar[stage], sa + kGAtom, col_a + 64, tok);
            for (int b = 0; b < nb; ++b)
              tma_load_2d(mb, &full_bar[stage], sa + kGStageA + b * kGAtom, is_a ? 64 * b : col_b, tok);
            if (++stage == stages) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_a = idesc_bf16(kGradBM, 64 * p.nb_a, true, true);
      constexpr uint32_t kIdescB = idesc_bf16(kGradBM, 64, true, true);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const int task = u / per_task;
        const bool is_a = u - task * per_task < p.units_a;
        const uint32_t idesc = is_a ? idesc_a : kIdescB;
        const uint64_t segs = p.task_segs[task];
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc) * kGAccStride;
        uint32_t accumulate = 0;
        for (int s = 0; s < p.num_segs; ++s) {
          if (!((segs >> s) & 1ull)) continue;
          for (int tok = so[s]; tok < so[s + 1]; tok += kGradBK) {
            const int nk = min(kGradBK, so[s + 1] - tok) / 16;
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a_base = smem_u32(pipe + stage * stage_bytes);
            const uint32_t b_base = a_base + kGStageA;
            for (int k = 0; k < nk; ++k) {
              const uint64_t ad = smem_desc(a_base + k * 16 * 128, kGAtom, 1024);
              const uint64_t bd = smem_desc(b_base + k * 16 * 128, kGAtom, 1024);
              mma_bf16(d_tmem, ad, bd, idesc, accumulate);
              accumulate = 1;
            }
            mma_commit(&empty_bar[stage]);
            if (++stage == stages) { stage = 0; phase ^= 1u; }
          }
        }
        mma_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      const int task = u / per_task;
      const int sub = u - task * per_task;
      const bool is_a = sub < p.units_a;
      const uint64_t segs = p.task_segs[task];
      bool any = false;
      for (int s = 0; s < p.num_segs; ++s)
        if (((segs >> s) & 1ull) && so[s + 1] > so[s]) any = true;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_addr =
          tmem_base + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(acc) * kGAccStride;
      uint32_t v0[32], v1[32];
      if (is_a) {
        // accumulator columns [s * r_cap, s * r_cap + rank_{t,s}) = dA_{t,s} rows (Gs column order)
        const int m = sub * kGradBM + 32 * q + lane;
        for (int sc = 0; sc < S; ++sc) {
          const int slot = task * S + sc;
          const int rank = p.slot_rank[slot];
          float* dA = p.slot_dA[slot];
          if (dA == nullptr) continue;
          for (int j0 = 0; j0 < rank; j0 += 16) {
            uint32_t v[16];
            tmem_ld16(t_addr + static_cast<uint32_t>(sc * p.r_cap + j0), v);
            tmem_ld_wait();
            if (m < p.K) {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (j0 + j < rank) dA[static_cast<size_t>(j0 + j) * p.K + m] = any ? __uint_as_float(v[j]) : 0.f;
            }
          }
        }
      } else {
        tmem_ld32(t_addr, v0);
        tmem_ld32(t_addr + 32, v1);
        tmem_ld_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (!is_a) {
        const int ub = sub - p.units_a;
        const int sc = b_slice(ub);
        const int slot = task * S + sc;
        const int rank = p.slot_rank[slot];
        const int m = (ub - p.b_units_off[sc]) * kGradBM + 32 * q + lane;   // row of dB_{t,s}
        float* dB = p.slot_dB[slot];
        if (dB != nullptr && m < p.slice_off[sc + 1] - p.slice_off[sc]) {
          float* row = dB + static_cast<size_t>(m) * rank;
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < rank) row[j] = any ? __uint_as_float(j < 32 ? v0[j & 31] : v1[j & 31]) : 0.f;
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kGradTmemCols>(tmem_base);
  }
}

cudaError_t launch_grad(const GradParams& p, int grid, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t ce = once_per_device(configured, [] {
    return cudaFuncSetAttribute(mux_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kGradSmemBytes));
  });
  if (ce != cudaSuccess) return ce;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGradThreads);
  cfg.dynamicSmemBytes = kGradSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mux_grad_kernel, p);
}

}  // namespace mux
