// racecheck_probe.cu — is compute-sanitizer racecheck's report on mux_gemm_kernel a tool artifact?
//
// A minimal, obviously race-free kernel with the fused GEMM's synchronisation pattern, nothing else:
// a ring of shared-memory stages, one elected thread of a producer warp refills a stage with a bulk
// async copy (cp.async.bulk global -> shared, completion counted on an mbarrier with expect_tx), the
// consumer warps wait on that mbarrier's phase, read the stage, then arrive on an "empty" mbarrier
// that the producer waits on before the next refill of the same stage.  Every access is ordered by
// mbarrier phases exactly as in gemm.cu (there the consumer is the tensor core, here plain loads, so
// the probe is even simpler).  If racecheck reports hazards here too — a write from the async proxy
// (no source location) against the ordered reads — its reports on the GEMM are the same artifact:
// racecheck does not model mbarrier complete_tx ordering of async-proxy writes.
// The result is checked on the host (every stage's sum), so the probe also proves the data is right.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -o racecheck_probe racecheck_probe.cu
// run:   compute-sanitizer --tool racecheck ./racecheck_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kStages = 4;
constexpr int kStageElems = 1024;          // 4 KB of int32 per stage
constexpr int kIters = 64;                 // refills
constexpr int kConsumers = 4;              // consumer warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void probe(const int* __restrict__ src, long long* __restrict__ sums) {
  __shared__ alignas(128) int stage[kStages][kStageElems];
  __shared__ uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {                       // producer
    if (lane == 0) {
      for (int i = 0; i < kIters; ++i) {
        const int s = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1u);   // consumers released this stage
        mbar_expect_tx(&full[s], kStageElems * 4);
        bulk_g2s(stage[s], src + static_cast<size_t>(i) * kStageElems, kStageElems * 4, &full[s]);
      }
    }
  } else {                               // consumers: warp w sums its quarter of every stage
    const int c = warp - 1;
    for (int i = 0; i < kIters; ++i) {
      const int s = i % kStages;
      const uint32_t ph = (i / kStages) & 1;
      mbar_wait(&full[s], ph);
      long long acc = 0;
      for (int j = c * (kStageElems / kConsumers) + lane; j < (c + 1) * (kStageElems / kConsumers); j += 32)
        acc += stage[s][j];
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      __syncwarp();
      if (lane == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&sums[i]), static_cast<unsigned long long>(acc));
        mbar_arrive(&empty[s]);
      }
    }
  }
}

// Second pattern: tcgen05.alloc writes the allocated TMEM address into shared memory (a write by the
// tensor-memory unit, not by an SM instruction); every thread reads it after the documented ordering
// tcgen05.fence::before_thread_sync -> bar.sync -> tcgen05.fence::after_thread_sync (gemm.cu does the
// same, with a cluster barrier).  racecheck's GEMM report is on exactly this slot (tmem_holder).
__global__ void probe_tmem(unsigned* out) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = holder;
  out[threadIdx.x] = base;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base) : "memory");
}

// Third: the GEMM's own form — a CTA pair (cluster of 2) allocating with tcgen05.alloc.cta_group::2
// from a warp of each CTA, then tcgen05.fence::before_thread_sync, bar.sync, barrier.cluster
// arrive/wait, tcgen05.fence::after_thread_sync, and every thread reads the address slot.
__global__ void __cluster_dims__(2, 1, 1) probe_tmem_pair(unsigned* out) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = holder;
  out[blockIdx.x * blockDim.x + threadIdx.x] = base;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(base) : "memory");
}

int main() {
  const size_t n = static_cast<size_t>(kIters) * kStageElems;
  int* h = new int[n];
  for (size_t i = 0; i < n; ++i) h[i] = static_cast<int>((i * 2654435761u) % 1000u);
  int* d;
  long long* ds;
  cudaMalloc(&d, n * 4);
  cudaMalloc(&ds, kIters * 8);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(ds, 0, kIters * 8);
  probe<<<1, 32 * (1 + kConsumers)>>>(d, ds);
  cudaError_t e = cudaDeviceSynchronize();
  long long got[kIters];
  cudaMemcpy(got, ds, sizeof(got), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < kIters; ++i) {
    long long want = 0;
    for (int j = 0; j < kStageElems; ++j) want += h[static_cast<size_t>(i) * kStageElems + j];
    bad += want != got[i];
  }
  printf("racecheck_probe: %s, %d of %d stage sums wrong\n", cudaGetErrorString(e), bad, kIters);
  unsigned* dt;
  unsigned ht[128];
  cudaMalloc(&dt, sizeof(ht));
  probe_tmem<<<1, 128>>>(dt);
  cudaError_t e2 = cudaDeviceSynchronize();
  cudaMemcpy(ht, dt, sizeof(ht), cudaMemcpyDeviceToHost);
  int same = 1;
  for (int i = 1; i < 128; ++i) same &= ht[i] == ht[0];
  printf("racecheck_probe tmem: %s, every thread read the same TMEM address: %s\n", cudaGetErrorString(e2),
         same ? "yes" : "no");
  unsigned* dp;
  unsigned hp[256];
  cudaMalloc(&dp, sizeof(hp));
  probe_tmem_pair<<<2, 128>>>(dp);
  cudaError_t e3 = cudaDeviceSynchronize();
  cudaMemcpy(hp, dp, sizeof(hp), cudaMemcpyDeviceToHost);
  int same2 = 1;
  for (int i = 1; i < 256; ++i) same2 &= hp[i] == hp[0];
  printf("racecheck_probe tmem pair: %s, every thread of both CTAs read the same TMEM address: %s\n",
         cudaGetErrorString(e3), same2 ? "yes" : "no");
  return bad != 0 || e != cudaSuccess || e2 != cudaSuccess || !same || e3 != cudaSuccess || !same2;
}
