// nvls.cu — tensor-parallel collectives reduced/broadcast INSIDE the NVSwitch
// (NVLink SHARP, "NVLS"): SURVEY §8(f) NEXT-1; the paper offloads the
// overlapped collectives to NVLink SHARP so that they need only ~8 CTAs
// (§3.4.2).  Every rank holds one copy of a symmetric buffer that
// is also bound to a multicast object (mux_nvls: uc_buf = this rank's copy,
// mc_buf = the multicast address; flags likewise).
//
//   reduce-scatter: each rank's GEMM writes its partial [world*rows, cols]
//     into its own copy (plain local stores); then on every rank a few CTAs
//     pull their own row block with multimem.ld_reduce — ONE load returns the
//     sum over all ranks' copies, reduced in the switch (fp32 accumulation,
//     .acc::f32) — and store it to `out`.
//   all-gather: each rank stores its rows once to the multicast address
//     (multimem.st): the switch writes them into every rank's copy.
//
// Synchronisation: per-call counters in the flag block, incremented on EVERY
// rank at once with multimem.red (release, system scope) and polled on the
// local copy (acquire): [0] RS partials ready, [1] RS reads done, [2] AG
// stores done, [3] AG buffer consumed (mux_nvls_release), [4] a local
// last-CTA counter.  After call `seq` on all ranks counter i = seq * world.
#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

struct NvlsParams {
  int world, rank, rows, cols;
  unsigned long long seq;
  const uint4* mc_buf;            // multicast address of [world * rows][cols] bf16
  unsigned long long* uc_flags;   // this rank's copy of the flag block
  unsigned long long* mc_flags;   // multicast address of the flag block
  uint4* out;                     // RS: [rows][cols] with row stride ldo8 uint4
  long long ldo8;
  const uint4* src;               // AG: this rank's rows [rows][cols], row stride lds8 uint4
  long long lds8;
  unsigned long long peer_wait_ns;
};

__device__ __forceinline__ void mm_red_add_release(unsigned long long* mc, unsigned long long v) {
  asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ uint4 mm_ld_reduce_bf16x8(const uint4* mc) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(mc)
               : "memory");
  return r;
}
__device__ __forceinline__ void mm_st_16B(const uint4* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void wait_counter(const unsigned long long* f, unsigned long long want,
                                             unsigned long long limit_ns) {
  if (ld_acquire_sys_u64(f) >= want) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys_u64(f) < want)
    if (peer_wait_expired(t0, limit_ns)) __trap();
}
// the last CTA of the grid to get here returns true (after every CTA's prior writes are fenced)
__device__ __forceinline__ bool last_cta(unsigned long long* ctr) {
  __threadfence_system();
  const unsigned long long n = atomicAdd(ctr, 1ull);
  if (n == gridDim.x - 1) {
    *ctr = 0ull;
    __threadfence_system();
    return true;
  }
  return false;
}

__global__ void __launch_bounds__(512) mux_nvls_rs_kernel(const __grid_constant__ NvlsParams p) {
  griddep_wait();             // this rank's partial (the GEMM before) is complete in its copy
  griddep_launch_dependents();
  const unsigned long long want = p.seq * static_cast<unsigned long long>(p.world);
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      __threadfence_system();
      mm_red_add_release(p.mc_flags + 0, 1ull);   // my partial is readable by every rank
    }
    wait_counter(p.uc_flags + 0, want, p.peer_wait_ns);   // every rank's partial is
  }
  __syncthreads();
  const int nc = p.cols / 8;
  const long long total = static_cast<long long>(p.rows) * nc;
  const uint4* base = p.mc_buf + static_cast<long long>(p.rank) * p.rows * nc;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / nc;
    const int c = static_cast<int>(i - r * nc);
    p.out[r * p.ldo8 + c] = mm_ld_reduce_bf16x8(base + i);
  }
  __syncthreads();
  if (threadIdx.x == 0 && last_cta(p.uc_flags + 4)) {
    mm_red_add_release(p.mc_flags + 1, 1ull);    // done reading every rank's copy
    // the next call's GEMM overwrites this rank's copy: every rank must be done reading it
    wait_counter(p.uc_flags + 1, want, p.peer_wait_ns);
  }
}

__global__ void __launch_bounds__(512) mux_nvls_ag_kernel(const __grid_constant__ NvlsParams p) {
  griddep_wait();
  griddep_launch_dependents();
  const unsigned long long w = static_cast<unsigned long long>(p.world);
  if (threadIdx.x == 0) wait_counter(p.uc_flags + 3, (p.seq - 1) * w, p.peer_wait_ns);  // previous call consumed
  __syncthreads();
  const int nc = p.cols / 8;
  const long long total = static_cast<long long>(p.rows) * nc;
  const uint4* dst = p.mc_buf + static_cast<long long>(p.rank) * p.rows * nc;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / nc;
    const int c = static_cast<int>(i - r * nc);
    mm_st_16B(dst + i, p.src[r * p.lds8 + c]);
  }
  __syncthreads();
  if (threadIdx.x == 0 && last_cta(p.uc_flags + 4)) {
    mm_red_add_release(p.mc_flags + 2, 1ull);    // my rows are in every rank's copy
    wait_counter(p.uc_flags + 2, p.seq * w, p.peer_wait_ns);   // and everyone's rows are in mine
  }
}

__global__ void mux_nvls_release_kernel(unsigned long long* mc_flags) {
  griddep_wait();
  griddep_launch_dependents();
  __threadfence_system();
  mm_red_add_release(mc_flags + 3, 1ull);
}

cudaError_t launch_nvls(const NvlsParams& p, int kind, int ctas, cudaStream_t s) {
  if (kind == 2) return launch_pdl(mux_nvls_release_kernel, dim3(1), dim3(32), 0, s, p.mc_flags);
  return launch_pdl(kind == 0 ? mux_nvls_rs_kernel : mux_nvls_ag_kernel, dim3(ctas), dim3(512), 0, s, p);
}

}  // namespace mux

// ---------------------------------------------------------------- C ABI
extern "C" {

size_t mux_nvls_flags_elems(void) { return 8; }

static mux_status nvls_check(const mux_nvls* nv, int32_t cols, int32_t ctas) {
  if (!nv || !nv->uc_buf || !nv->mc_buf || !nv->uc_flags || !nv->mc_flags)
    return mux_set_error(MUX_ERR_INVALID_ARGUMENT, "nvls: null buffer or flag pointer");
  if (nv->world < 1 || nv->world > MUX_RS_MAX_WORLD || nv->rank < 0 || nv->rank >= nv->world || nv->seq == 0 ||
      nv->rows_per_rank <= 0 || cols < 8 || cols % 8 || ctas < 0 || ctas > 1024)
    return mux_set_error(MUX_ERR_INVALID_ARGUMENT, "nvls: world/rank/seq/rows/cols/ctas out of range");
  if ((reinterpret_cast<uintptr_t>(nv->uc_buf) | reinterpret_cast<uintptr_t>(nv->mc_buf)) & 15u)
    return mux_set_error(MUX_ERR_INVALID_ARGUMENT, "nvls: buffers must be 16-byte aligned");
  return MUX_OK;
}

static mux::NvlsParams nvls_params(const mux_nvls* nv, int32_t cols) {
  mux::NvlsParams p{};
  p.world = nv->world;
  p.rank = nv->rank;
  p.rows = nv->rows_per_rank;
  p.cols = cols;
  p.seq = nv->seq;
  p.mc_buf = reinterpret_cast<const uint4*>(nv->mc_buf);
  p.uc_flags = nv->uc_flags;
  p.mc_flags = nv->mc_flags;
  p.peer_wait_ns = mux_peer_wait_ns();
  return p;
}

mux_status mux_nvls_reduce_scatter(const mux_nvls* nv, int32_t cols, mux_bf16* out, int64_t ldo, int32_t ctas,
                                   cudaStream_t stream) {
  mux_status st = nvls_check(nv, cols, ctas);
  if (st != MUX_OK) return st;
  if (!out || (reinterpret_cast<uintptr_t>(out) & 15u) || ldo < cols || ldo % 8)
    return mux_set_error(MUX_ERR_INVALID_ARGUMENT, "nvls_reduce_scatter: out null/misaligned or ldo < cols");
  mux::NvlsParams p = nvls_params(nv, cols);
  p.out = reinterpret_cast<uint4*>(out);
  p.ldo8 = ldo / 8;
  cudaError_t e = mux::launch_nvls(p, 0, ctas ? ctas : 16, stream);
  return e == cudaSuccess ? MUX_OK : mux_set_error(MUX_ERR_CUDA, cudaGetErrorString(e));
}

mux_status mux_nvls_all_gather(const mux_nvls* nv, const mux_bf16* rows, int64_t ld, int32_t cols, int32_t ctas,
                               cudaStream_t stream) {
  mux_status st = nvls_check(nv, cols, ctas);
  if (st != MUX_OK) return st;
  if (!rows || (reinterpret_cast<uintptr_t>(rows) & 15u) || ld < cols || ld % 8)
    return mux_set_error(MUX_ERR_INVALID_ARGUMENT, "nvls_all_gather: rows null/misaligned or ld < cols");
  mux::NvlsParams p = nvls_params(nv, cols);
  p.src = reinterpret_cast<const uint4*>(rows);
  p.lds8 = ld / 8;
  cudaError_t e = mux::launch_nvls(p, 1, ctas ? ctas : 16, stream);
  return e == cudaSuccess ? MUX_OK : mux_set_error(MUX_ERR_CUDA, cudaGetErrorString(e));
}

mux_status mux_nvls_release(const mux_nvls* nv, cudaStream_t stream) {
  if (!nv || !nv->mc_flags) return mux_set_error(MUX_ERR_INVALID_ARGUMENT, "nvls_release: null flags");
  mux::NvlsParams p{};
  p.mc_flags = nv->mc_flags;
  cudaError_t e = mux::launch_nvls(p, 2, 1, stream);
  return e == cudaSuccess ? MUX_OK : mux_set_error(MUX_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
