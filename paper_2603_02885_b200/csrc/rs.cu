// rs.cu — the receive side of the fused GEMM -> reduce-scatter (tensor
// parallelism; NEXT-1's "GEMM epilogue -> peer NVLink stores").
// The fused GEMM of every rank s writes its partial output tile by tile
// straight into the receive slot s of the rank that owns the tile's rows
// (mux_linear_fwd_rs / mux_linear_bwd_dx_rs); this kernel, on the owner rank,
// waits for the ready flags of all sources, sums the `world` partial slots in
// fp32 (fixed ascending source order: deterministic) and acknowledges every
// source so it may overwrite its slot on the next call.
//
// Flag block of rank d (zeroed once): [0, world) ready (source s writes seq),
// [world, 2 world) ack (rank s writes seq after reducing), [2 world] a local
// completion counter of this kernel.
#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {


__global__ void __launch_bounds__(256) mux_rs_reduce_kernel(const __grid_constant__ RsReduceParams p) {
  griddep_wait();
  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.world; ++s) {
      const unsigned long long* f = p.flags + s;
      if (ld_acquire_sys_u64(f) < p.seq) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_sys_u64(f) < p.seq)
          if (peer_wait_expired(t0, p.peer_wait_ns)) __trap();
      }
    }
  }
  __syncthreads();
  const int nc = p.cols / 8;
  const long long total = static_cast<long long>(p.rows) * nc;
  const long long slot = total;  // uint4 per slot
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < p.world; ++s) {
      const uint4 v = p.recv[s * slot + i];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[2 * e] += __uint_as_float(w[e] << 16);
        acc[2 * e + 1] += __uint_as_float(w[e] & 0xFFFF0000u);
      }
    }
    const long long r = i / nc;
    const int c = static_cast<int>(i - r * nc);
    p.out[r * p.ldo8 + c] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                       pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
  }
  // the last block to finish acknowledges every source (its slot may be rewritten)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned long long* ctr = p.flags + 2 * p.world;
    if (atomicAdd(ctr, 1ull) == gridDim.x - 1) {
      *ctr = 0ull;
      __threadfence_system();
      for (int s = 0; s < p.world; ++s) st_release_sys_u64(p.ack[s], p.seq);
    }
  }
}

cudaError_t launch_rs_reduce(const RsReduceParams& p, int num_sms, cudaStream_t s) {
  const long long work = static_cast<long long>(p.rows) * (p.cols / 8);
  long long blocks = (work + 255) / 256;
  if (blocks > num_sms * 4LL) blocks = num_sms * 4LL;
  if (blocks < 1) blocks = 1;
  return launch_pdl(mux_rs_reduce_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, p);
}

}  // namespace mux
