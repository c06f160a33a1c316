// gemm.cu — fused multiplexed-LoRA linear for sm_100a (tcgen05 + TMEM + TMA).
//
// One persistent, warp-specialized kernel computes, for all segments of an
// hTask at once (spatial batching of the BaseOp, Eq. 1 P:484-489 / Eq. 2
// P:491-498) plus every segment's LoRA adapter (north_star formula), fused
// horizontally across tasks:
//
//   fwd:  Y  = X W^T            + Hs B_t^T      Hs = bf16(s_t X A_t^T)
//   bwd:  dX = dY W             + Gs A_t        Gs = bf16(s_t dY B_t)
//
// Work items ("tiles"), statically round-robined over a grid of #SMs CTAs:
//   * side tiles  (one per 128-row block m): the shrink Hs/Gs[m] = s_t X_m A_t^T
//     as a tcgen05 MMA with N = 64 (rank padded), written to global and
//     published through flags[m];
//   * main tiles  (m, n): the backbone product over the whole reduction, then
//     one "extension" k-block per task present in the tile: A = Hs/Gs tile,
//     B = B_t / A_t tile (the expand), accumulated into the same TMEM tile.
// Segments are multiples of 64 rows, so a 128-row tile holds at most two
// tasks; their adapter MMAs use the disable-output-lane mask so that a row is
// only ever multiplied with its own task's weights (NaN isolation).
// Side tiles come first in the schedule and never wait, so every main tile's
// dependency is on a lower-indexed tile: with all CTAs resident the smallest
// unfinished tile can always progress (no deadlock).
//
// Roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 =
// TMEM allocator, warps 4..7 = epilogue (TMEM -> regs -> bf16 -> smem ->
// TMA store).  4-stage smem ring (48 KB/stage), 2 TMEM accumulators of 256
// fp32 columns so the epilogue of tile i overlaps the mainloop of tile i+1.
#include "common.h"
#include "ptx.cuh"

namespace mux {

constexpr uint32_t kStageA = kBM * kBK * 2;          // 16 KB
constexpr uint32_t kSubB = 64 * kBK * 2;             // 8 KB: one {64 x 128 B} TMA box
constexpr uint32_t kStageB = kBN * kBK * 2;          // 32 KB
constexpr uint32_t kStageBytes = kStageA + kStageB;  // 48 KB
constexpr uint32_t kEpiBuf = 32 * 128;               // 32 rows x 64 bf16 (one TMA store box)
constexpr uint32_t kSmemPipe = kStages * kStageBytes;
constexpr uint32_t kSmemEpi = 4 * 2 * kEpiBuf;
constexpr uint32_t kSmemMisc = 1024;
constexpr uint32_t kGemmSmemBytes = kSmemPipe + kSmemEpi + kSmemMisc + 1024;
constexpr uint32_t kTmemCols = 512;
constexpr int kGemmThreads = 256;
constexpr int kGroupM = 8;  // raster: 8 row-blocks share a band of W tiles

struct TileGroups {
  int n;          // active groups (tasks with rank > 0) in the tile
  int seg0, seg1;
  int half0, half1;  // lanes the group owns: 0 = all 128, 1 = rows 0-63, 2 = rows 64-127
};

// disable-output-lane mask word w (lanes 32w..32w+31) for a group owning `half`
__device__ __forceinline__ uint32_t lane_mask(int half, int w) {
  return half == 0 ? 0u : (half == 1 ? (w >= 2 ? ~0u : 0u) : (w < 2 ? ~0u : 0u));
}

__device__ __forceinline__ int seg_containing(const int* so, int S, int row) {
  for (int s = 0; s < S; ++s)
    if (so[s] <= row && row < so[s + 1]) return s;
  return -1;
}

__device__ __forceinline__ TileGroups tile_groups(const GemmParams& p, const int* so, int m) {
  TileGroups g;
  g.n = 0;
  g.seg0 = g.seg1 = 0;
  g.half0 = g.half1 = 0;
  const int S = p.num_segs;
  const int r0 = m * kBM;
  const int s0 = seg_containing(so, S, r0);
  const int s1 = seg_containing(so, S, r0 + kRowHalf);
  if (s1 < 0 || s1 == s0) {
    if (s0 >= 0 && p.seg_rank[s0] > 0) {
      g.seg0 = s0;
      g.half0 = 0;
      g.n = 1;
    }
  } else {
    if (s0 >= 0 && p.seg_rank[s0] > 0) {
      g.seg0 = s0;
      g.half0 = 1;
      g.n = 1;
    }
    if (p.seg_rank[s1] > 0) {
      if (g.n == 0) { g.seg0 = s1; g.half0 = 2; }
      else { g.seg1 = s1; g.half1 = 2; }
      ++g.n;
    }
  }
  return g;
}

struct Tile {
  int m, n;
  bool side;
};

__device__ __forceinline__ Tile tile_at(int t, int num_m, int num_n) {
  Tile r;
  if (t < num_m) {
    r.m = t; r.n = 0; r.side = true;
    return r;
  }
  const int v = t - num_m;
  const int per_group = kGroupM * num_n;
  const int grp = v / per_group;
  const int first_m = grp * kGroupM;
  const int gm = min(num_m - first_m, kGroupM);
  const int w = v - grp * per_group;
  r.m = first_m + w % gm;
  r.n = w / gm;
  r.side = false;
  return r;
}

template <bool kBwd>
__global__ void __launch_bounds__(kGemmThreads, 1) mux_gemm_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* pipe = smem;
  uint8_t* epi = smem + kSmemPipe;
  uint8_t* misc = epi + kSmemEpi;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(misc);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* so = reinterpret_cast<int*>(misc + 256);  // seg_off copy, <= 65 ints

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i <= p.num_segs; i += blockDim.x) so[i] = p.seg_off[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.map_a);
    tma_prefetch(&p.map_w);
    tma_prefetch(&p.map_side);
    tma_prefetch(&p.map_out);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total_rows = so[p.num_segs];
  const int num_m = (total_rows + kBM - 1) / kBM;
  const int num_n = (p.nout + kBN - 1) / kBN;
  const int total_tiles = num_m * (1 + (p.has_main ? num_n : 0));
  const int num_kb = p.kred / kBK;

  if (warp == 0) {
    // =========================== TMA producer ===========================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto advance = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      };
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const Tile tl = tile_at(t, num_m, num_n);
        const TileGroups g = tile_groups(p, so, tl.m);
        const int row0 = tl.m * kBM;
        if (tl.side) {
          if (g.n == 0) continue;
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1u);
            uint8_t* sa = pipe + stage * kStageBytes;
            uint8_t* sb = sa + kStageA;
            mbar_arrive_expect_tx(&full_bar[stage], kStageA + g.n * kSubB);
            tma_load_2d(&p.map_a, &full_bar[stage], sa, kb * kBK, row0);
            for (int i = 0; i < g.n; ++i) {
              const int ad = p.seg_adapter[i == 0 ? g.seg0 : g.seg1];
              if (!kBwd)  // A_t [r, K] K-major: box {64 k, 64 j}
                tma_load_2d(&p.map_lora_a[ad], &full_bar[stage], sb + i * kSubB, kb * kBK, 0);
              else        // B_t [N, r] as MN-major {64 j, 64 n}
                tma_load_2d(&p.map_lora_b[ad], &full_bar[stage], sb + i * kSubB, 0, kb * kBK);
            }
            advance();
          }
        } else {
          const int col0 = tl.n * kBN;
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1u);
            uint8_t* sa = pipe + stage * kStageBytes;
            uint8_t* sb = sa + kStageA;
            mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
            tma_load_2d(&p.map_a, &full_bar[stage], sa, kb * kBK, row0);
            for (int i = 0; i < 4; ++i) {
              if (!kBwd)  // W [N, K] K-major rows n
                tma_load_2d(&p.map_w, &full_bar[stage], sb + i * kSubB, kb * kBK, col0 + 64 * i);
              else        // W viewed [k_out (MN), n (red)]: MN-major atoms of 64 k
                tma_load_2d(&p.map_w, &full_bar[stage], sb + i * kSubB, col0 + 64 * i, kb * kBK);
            }
            advance();
          }
          if (g.n > 0) {
            // wait until the side tile of this row block has published Hs/Gs
            const int* flag = p.flags + tl.m;
            if (ld_acquire_gpu(flag) < 4) {
              const uint64_t t0 = globaltimer_ns();
              while (ld_acquire_gpu(flag) < 4) {
                if (globaltimer_ns() - t0 > kWatchdogNs) __trap();
              }
            }
            fence_async_global();
          }
          for (int i = 0; i < g.n; ++i) {
            const int ad = p.seg_adapter[i == 0 ? g.seg0 : g.seg1];
            mbar_wait(&empty_bar[stage], phase ^ 1u);
            uint8_t* sa = pipe + stage * kStageBytes;
            uint8_t* sb = sa + kStageA;
            mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
            tma_load_2d(&p.map_side, &full_bar[stage], sa, 0, row0);
            for (int j = 0; j < 4; ++j) {
              if (!kBwd)  // B_t [N, r] K-major rows n: box {64 j, 64 n}
                tma_load_2d(&p.map_lora_b[ad], &full_bar[stage], sb + j * kSubB, 0, col0 + 64 * j);
              else        // A_t [r, K] viewed [k_out (MN), j (red)]
                tma_load_2d(&p.map_lora_a[ad], &full_bar[stage], sb + j * kSubB, col0 + 64 * j, 0);
            }
            advance();
          }
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer =============================
    if (lane == 0) {
      constexpr uint32_t kIdescMain = idesc_bf16(kBM, kBN, false, kBwd);
      constexpr uint32_t kIdescSide = idesc_bf16(kBM, kSideN, false, kBwd);
      // B-operand descriptor parameters: K-major rows of 128 B (SBO 1024) or
      // MN-major atoms of 64 elements x 64 K-rows (LBO 8 KB, SBO 1024).
      constexpr uint32_t kBLbo = kBwd ? kSubB : 16;
      constexpr uint32_t kBStepK = kBwd ? 16 * 128 : 32;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      auto advance = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      };
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const Tile tl = tile_at(t, num_m, num_n);
        const TileGroups g = tile_groups(p, so, tl.m);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
        if (tl.side) {
          if (g.n > 0) {
            for (int kb = 0; kb < num_kb; ++kb) {
              mbar_wait(&full_bar[stage], phase);
              tc_fence_after();
              const uint32_t a_base = smem_u32(pipe + stage * kStageBytes);
              const uint32_t b_base = a_base + kStageA;
              for (int i = 0; i < g.n; ++i) {
                const int half = i == 0 ? g.half0 : g.half1;
                const uint32_t m0 = lane_mask(half, 0), m1 = lane_mask(half, 1);
                const uint32_t m2 = lane_mask(half, 2), m3 = lane_mask(half, 3);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                  const uint64_t ad = smem_desc(a_base + k * 32, 16, 1024);
                  const uint64_t bd = smem_desc(b_base + i * kSubB + k * kBStepK, kBLbo, 1024);
                  mma_bf16_masked(d_tmem, ad, bd, kIdescSide, (kb | k) != 0, m0, m1, m2, m3);
                }
              }
              mma_commit(&empty_bar[stage]);
              advance();
            }
          }
        } else {
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a_base = smem_u32(pipe + stage * kStageBytes);
            const uint32_t b_base = a_base + kStageA;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t ad = smem_desc(a_base + k * 32, 16, 1024);
              const uint64_t bd = smem_desc(b_base + k * kBStepK, kBLbo, 1024);
              mma_bf16(d_tmem, ad, bd, kIdescMain, (kb | k) != 0);
            }
            mma_commit(&empty_bar[stage]);
            advance();
          }
          for (int i = 0; i < g.n; ++i) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a_base = smem_u32(pipe + stage * kStageBytes);
            const uint32_t b_base = a_base + kStageA;
            const int nk = (p.seg_rank[i == 0 ? g.seg0 : g.seg1] + 15) / 16;
            const int half = i == 0 ? g.half0 : g.half1;
            const uint32_t m0 = lane_mask(half, 0), m1 = lane_mask(half, 1);
            const uint32_t m2 = lane_mask(half, 2), m3 = lane_mask(half, 3);
            for (int k = 0; k < nk; ++k) {
              const uint64_t ad = smem_desc(a_base + k * 32, 16, 1024);
              const uint64_t bd = smem_desc(b_base + k * kBStepK, kBLbo, 1024);
              mma_bf16_masked(d_tmem, ad, bd, kIdescMain, 1u, m0, m1, m2, m3);
            }
            mma_commit(&empty_bar[stage]);
            advance();
          }
        }
        mma_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  } else if (warp >= 4) {
    // =========================== epilogue ===============================
    const int q = warp & 3;  // TMEM lane quadrant = rows 32q .. 32q+31
    int acc = 0;
    uint32_t acc_phase = 0;
    uint8_t* bufs = epi + q * 2 * kEpiBuf;
    int buf_sel = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const Tile tl = tile_at(t, num_m, num_n);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row_w = tl.m * kBM + 32 * q;  // first row of this warp
      const uint32_t t_addr = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(acc * kBN);
      if (tl.side) {
        uint32_t v0[32], v1[32];
        tmem_ld32(t_addr, v0);
        tmem_ld32(t_addr + 32, v1);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        const int row = row_w + lane;
        if (row < total_rows) {
          const int s = seg_containing(so, p.num_segs, row);
          const int rank = s >= 0 ? p.seg_rank[s] : 0;
          const float sc = s >= 0 ? p.seg_scale[s] : 0.f;
          uint4* dst = reinterpret_cast<uint4*>(p.side_out + static_cast<size_t>(row) * p.r_cap);
#pragma unroll
          for (int j0 = 0; j0 < 64; j0 += 8) {
            if (j0 < p.r_cap) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int j = j0 + 2 * e;
                const uint32_t a = j < 32 ? v0[j & 31] : v1[j & 31];
                const uint32_t b = j + 1 < 32 ? v0[(j + 1) & 31] : v1[(j + 1) & 31];
                const float lo = j < rank ? __uint_as_float(a) * sc : 0.f;
                const float hi = j + 1 < rank ? __uint_as_float(b) * sc : 0.f;
                w[e] = pack_bf16x2(lo, hi);
              }
              dst[j0 / 8] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        fence_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) red_release_gpu_add(p.flags + tl.m, 1);
      } else {
        const bool valid = row_w < total_rows;
        const int col_t = tl.n * kBN;
#pragma unroll 1
        for (int c = 0; c < kBN / 64; ++c) {
          uint32_t v0[32], v1[32];
          tmem_ld32(t_addr + c * 64, v0);
          tmem_ld32(t_addr + c * 64 + 32, v1);
          tmem_ld_wait();
          if (c == kBN / 64 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[acc]);
          }
          uint8_t* buf = bufs + buf_sel * kEpiBuf;
          if (lane == 0) tma_store_wait_read<1>();
          __syncwarp();
          uint8_t* rowp = buf + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint32_t* v = ch < 4 ? v0 : v1;
            const int b = (ch & 3) * 8;
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(v[b + 0]), __uint_as_float(v[b + 1]));
            w.y = pack_bf16x2(__uint_as_float(v[b + 2]), __uint_as_float(v[b + 3]));
            w.z = pack_bf16x2(__uint_as_float(v[b + 4]), __uint_as_float(v[b + 5]));
            w.w = pack_bf16x2(__uint_as_float(v[b + 6]), __uint_as_float(v[b + 7]));
            *reinterpret_cast<uint4*>(rowp + ((ch ^ (lane & 7)) << 4)) = w;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            const int col = col_t + c * 64;
            if (valid && col < p.nout) tma_store_2d(&p.map_out, buf, col, row_w);
            tma_store_commit();
          }
          buf_sel ^= 1;
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    if (lane == 0) tma_store_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------- launchers
template <bool kBwd>
cudaError_t launch_gemm_impl(const GemmParams& p, int grid, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(mux_gemm_kernel<kBwd>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kGemmSmemBytes));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  mux_gemm_kernel<kBwd><<<grid, kGemmThreads, kGemmSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmParams& p, bool bwd, int grid, cudaStream_t stream) {
  return bwd ? launch_gemm_impl<true>(p, grid, stream) : launch_gemm_impl<false>(p, grid, stream);
}

}  // namespace mux
