// launch.cuh — kernel launch with programmatic dependent launch (PDL): every
// kernel of the library starts with griddepcontrol.wait, so its launch and
// prologue overlap the tail of the previous kernel on the stream.
#pragma once
#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

namespace mux {

// Function attributes (dynamic smem size, carveout) are per device: `setup`
// runs (idempotently) the first time each device launches the kernel; safe
// under concurrent first calls from several host threads.
template <typename F>
cudaError_t once_per_device(std::atomic<uint64_t>& done, F setup) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = setup();
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace mux
