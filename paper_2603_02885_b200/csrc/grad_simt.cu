// grad_simt.cu — segmented adapter-weight gradients on the CUDA cores (sm_100a).
//
// Same operation, operands and work units as grad.cu (dA_t = Σ_i Gs[i,:]ᵀ X[i,:],
// dB_t = Σ_i dY[i,:]ᵀ Hs[i,:], P:491-499 chain rule, reductions over the
// task's tokens), computed with warp-level FMAs instead of tcgen05:
// north_star asks for "warp-level reductions where rank is too small for tensor
// cores", and this kernel is the measured alternative (A/B in DESIGN §6.2).
//
// Producer: one warp streams the same TMA tiles as grad.cu (128 tokens x 128
// output columns of X / dY, 128 tokens x 64 rank columns of Gs / Hs, 128 B
// swizzle) through a ring of kSimtStages stages.  Consumers: 16 warps; thread
// (column pair cp, group q) accumulates an outer product of 2 columns x JPT
// ranks in fp32 registers over the tokens of its token group (tokens
// i ≡ tg mod NTG); the NTG token-group partials are then summed in smem in
// ascending group order (deterministic; one owner per output element).
//   rank <= 4: JPT 4, NTG 8   rank <= 8: JPT 4, NTG 4   rank <= 16: JPT 4, NTG 2
//   rank <= 32: JPT 8, NTG 2  rank <= 64: JPT 16, NTG 2
// ALU cost per token and thread: one 4-byte X load, JPT/8 16-byte rank loads
// (broadcast), 2 + JPT bf16->fp32 widenings and 2·JPT FFMAs.
#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

namespace {

constexpr uint32_t kSAtom = kGradBK * 128;          // 128 token rows x 128 B = 16 KB
constexpr uint32_t kSStageA = 2 * kSAtom;           // 128 output columns
constexpr uint32_t kSStageBytes = kSStageA + kSAtom;  // + 64 rank columns = 48 KB
constexpr int kSimtStages = 3;
constexpr int kSimtConsumers = 512;                 // 16 warps
constexpr int kSimtThreads = kSimtConsumers + 32;   // + producer warp
constexpr uint32_t kSimtRedBytes = 32u * kSimtConsumers * 4u;  // up to 2 x 16 partials per thread
constexpr uint32_t kSimtSmemBytes = kSimtStages * kSStageBytes + kSimtRedBytes + 1024 + 1024;

__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kSimtConsumers)); }

__device__ __forceinline__ float lo_f(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_f(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// One unit: (task, 128 output columns).  Consumes the stages the producer
// loaded for it (same order), then reduces and writes its outputs.
template <int JPT, int NTG>
__device__ __forceinline__ void simt_unit(const GradParams& p, const uint8_t* pipe, uint64_t* full_bar,
                                          uint64_t* empty_bar, float* red, const int* so, int& stage,
                                          uint32_t& phase, int task, bool is_a, int m0) {
  constexpr int QPG = 8 / NTG;  // rank groups per token group
  const int ctid = threadIdx.x;
  const int cp = ctid & 63;
  const int q = ctid >> 6;
  const int tg = q / QPG;
  const int j0 = (q % QPG) * JPT;
  const int lane = ctid & 31;
  const uint32_t xoff = static_cast<uint32_t>(cp >> 5) * kSAtom + static_cast<uint32_t>((cp & 3) << 2);
  const uint32_t xchunk = static_cast<uint32_t>((cp & 31) >> 2);
  const uint32_t gchunk = static_cast<uint32_t>(j0 >> 3);
  const uint32_t gin = static_cast<uint32_t>((j0 & 7) * 2);
  float acc[2][JPT];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int j = 0; j < JPT; ++j) acc[c][j] = 0.f;

  const uint64_t segs = p.task_segs[task];
  for (int s = 0; s < p.num_segs; ++s) {
    if (!((segs >> s) & 1ull)) continue;
    for (int tok = so[s]; tok < so[s + 1]; tok += kGradBK) {
      const int nvalid = min(kGradBK, so[s + 1] - tok);
      mbar_wait(&full_bar[stage], phase);
      const uint8_t* sx = pipe + stage * kSStageBytes;
      const uint8_t* sg = sx + kSStageA;
      if (j0 < p.r_cap) {
#pragma unroll 4
        for (int i = tg; i < nvalid; i += NTG) {
          const uint32_t sw = static_cast<uint32_t>(i & 7);
          const uint32_t xw = *reinterpret_cast<const uint32_t*>(sx + xoff + i * 128 + ((xchunk ^ sw) << 4));
          const float x0 = lo_f(xw), x1 = hi_f(xw);
          uint32_t gw[JPT / 2];
          if constexpr (JPT == 4) {
            const uint2 v = *reinterpret_cast<const uint2*>(sg + i * 128 + ((gchunk ^ sw) << 4) + gin);
            gw[0] = v.x;
            gw[1] = v.y;
          } else {
#pragma unroll
            for (int h = 0; h < JPT / 8; ++h) {
              const uint4 v =
                  *reinterpret_cast<const uint4*>(sg + i * 128 + (((gchunk + h) ^ sw) << 4));
              gw[4 * h + 0] = v.x;
              gw[4 * h + 1] = v.y;
              gw[4 * h + 2] = v.z;
              gw[4 * h + 3] = v.w;
            }
          }
#pragma unroll
          for (int h = 0; h < JPT / 2; ++h) {
            const float g0 = lo_f(gw[h]), g1 = hi_f(gw[h]);
            acc[0][2 * h] = fmaf(x0, g0, acc[0][2 * h]);
            acc[0][2 * h + 1] = fmaf(x0, g1, acc[0][2 * h + 1]);
            acc[1][2 * h] = fmaf(x1, g0, acc[1][2 * h]);
            acc[1][2 * h + 1] = fmaf(x1, g1, acc[1][2 * h + 1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[stage]);
      if (++stage == kSimtStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  }

  // token-group partials -> group 0, ascending group order
  if (NTG > 1) {
    if (tg > 0) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int j = 0; j < JPT; ++j) red[(c * JPT + j) * kSimtConsumers + ctid] = acc[c][j];
    }
    consumers_sync();
    if (tg == 0) {
      for (int g = 1; g < NTG; ++g) {
        const int src = ctid + g * QPG * 64;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int j = 0; j < JPT; ++j) acc[c][j] += red[(c * JPT + j) * kSimtConsumers + src];
      }
    }
    consumers_sync();
  }
  if (tg != 0) return;
  const int rank = p.task_rank[task];
  if (is_a) {
    float* dA = p.task_dA[task];
    if (dA == nullptr) return;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int k = m0 + 2 * cp + c;
      if (k >= p.K) continue;
#pragma unroll
      for (int j = 0; j < JPT; ++j)
        if (j0 + j < rank) dA[static_cast<size_t>(j0 + j) * p.K + k] = acc[c][j];
    }
  } else {
    float* dB = p.task_dB[task];
    if (dB == nullptr) return;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int n = m0 + 2 * cp + c;
      if (n >= p.N) continue;
      float* row = dB + static_cast<size_t>(n) * rank;
#pragma unroll
      for (int j = 0; j < JPT; ++j)
        if (j0 + j < rank) row[j0 + j] = acc[c][j];
    }
  }
}

__global__ void __launch_bounds__(kSimtThreads, 1) mux_grad_simt_kernel(const __grid_constant__ GradParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* pipe = smem;
  float* red = reinterpret_cast<float*>(smem + kSimtStages * kSStageBytes);
  uint8_t* misc = smem + kSimtStages * kSStageBytes + kSimtRedBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(misc);
  uint64_t* empty_bar = full_bar + kSimtStages;
  int* so = reinterpret_cast<int*>(misc + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kProducerWarp = kSimtConsumers / 32;
  if (warp == kProducerWarp && lane == 0) {
    tma_prefetch(&p.map_x);
    tma_prefetch(&p.map_dy);
    tma_prefetch(&p.map_hs);
    tma_prefetch(&p.map_gs);
    for (int s = 0; s < kSimtStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kSimtConsumers / 32);
    }
    fence_mbar_init();
  }
  griddep_wait();  // PDL: the prologue above overlaps the previous kernel
  griddep_launch_dependents();
  for (int i = threadIdx.x; i <= p.num_segs; i += blockDim.x) so[i] = p.seg_off[i];
  __syncthreads();

  const int per_task = p.units_a + p.units_b;
  const int total_units = p.num_tasks * per_task;
  if (warp == kProducerWarp) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const int task = u / per_task;
        const int sub = u - task * per_task;
        const bool is_a = sub < p.units_a;
        const int m0 = (is_a ? sub : sub - p.units_a) * kGradBM;
        const CUtensorMap* ma = is_a ? &p.map_x : &p.map_dy;
        const CUtensorMap* mb = is_a ? &p.map_gs : &p.map_hs;
        const uint64_t segs = p.task_segs[task];
        for (int s = 0; s < p.num_segs; ++s) {
          if (!((segs >> s) & 1ull)) continue;
          for (int tok = so[s]; tok < so[s + 1]; tok += kGradBK) {
            mbar_wait(&empty_bar[stage], phase ^ 1u);
            uint8_t* sa = pipe + stage * kSStageBytes;
            mbar_arrive_expect_tx(&full_bar[stage], kSStageBytes);
            tma_load_2d(ma, &full_bar[stage], sa, m0, tok);
            tma_load_2d(ma, &full_bar[stage], sa + kSAtom, m0 + 64, tok);
            tma_load_2d(mb, &full_bar[stage], sa + kSStageA, 0, tok);
            if (++stage == kSimtStages) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
    return;
  }
  int stage = 0;
  uint32_t phase = 0;
  for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
    const int task = u / per_task;
    const int sub = u - task * per_task;
    const bool is_a = sub < p.units_a;
    const int m0 = (is_a ? sub : sub - p.units_a) * kGradBM;
    const int rank = p.task_rank[task];
    if (rank <= 4)
      simt_unit<4, 8>(p, pipe, full_bar, empty_bar, red, so, stage, phase, task, is_a, m0);
    else if (rank <= 8)
      simt_unit<4, 4>(p, pipe, full_bar, empty_bar, red, so, stage, phase, task, is_a, m0);
    else if (rank <= 16)
      simt_unit<4, 2>(p, pipe, full_bar, empty_bar, red, so, stage, phase, task, is_a, m0);
    else if (rank <= 32)
      simt_unit<8, 2>(p, pipe, full_bar, empty_bar, red, so, stage, phase, task, is_a, m0);
    else
      simt_unit<16, 2>(p, pipe, full_bar, empty_bar, red, so, stage, phase, task, is_a, m0);
  }
}

}  // namespace

cudaError_t launch_grad_simt(const GradParams& p, int grid, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t ce = once_per_device(configured, [] {
    return cudaFuncSetAttribute(mux_grad_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSimtSmemBytes));
  });
  if (ce != cudaSuccess) return ce;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSimtThreads);
  cfg.dynamicSmemBytes = kSimtSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mux_grad_simt_kernel, p);
}

}  // namespace mux
