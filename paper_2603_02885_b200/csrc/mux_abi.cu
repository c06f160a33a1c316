// mux_abi.cu — the C ABI of libmux (include/mux.h): host-side validation,
// workspace carving, TMA descriptor encoding and kernel launches.  Every
// entry point only enqueues on the caller's stream; nothing reads device
// data on the host, so whole layers can be captured in a CUDA graph.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include <cuda.h>
#include <cuda_runtime.h>

// fused GEMM: outputs this narrow use 256 x 128 tiles (only where a 256-wide tile would be at least
// half empty: wider narrow tiles lose more to the doubled A-operand feed than they gain in balance,
// profiles/r01_gemm_ab_narrow.jsonl)
#ifndef MUX_NARROW_MAX_NOUT
#define MUX_NARROW_MAX_NOUT 128
#endif
// fused GEMM: outputs at least this wide use 256 x 512 pair tiles (gemm.cu kTileN = 512)
#ifndef MUX_WIDE_MIN_NOUT
#define MUX_WIDE_MIN_NOUT (1 << 30)
#endif
// fused GEMM: reductions this short schedule every shrink tile before the main tiles
#ifndef MUX_SIDE_FIRST_MAX_KRED
#define MUX_SIDE_FIRST_MAX_KRED 2048
#endif

#include "common.h"

namespace mux {
cudaError_t launch_gemm(const GemmParams& p, bool bwd, int tile_n, int grid, cudaStream_t stream);
cudaError_t launch_grad(const GradParams& p, int grid, cudaStream_t stream);
cudaError_t launch_grad_simt(const GradParams& p, int grid, cudaStream_t stream);
size_t pack_workspace_bytes(int M, int S);
cudaError_t launch_pack(int M, int S, const int32_t* task_seq_off, const int32_t* seq_len,
                        const int32_t* pack_capacity, int chunk_size, int chunk_min, int max_rows, int max_chunks,
                        int32_t* seg_off, int32_t* seq_row, int32_t* chunk_task, int32_t* chunk_pack,
                        int32_t* chunk_valid, int32_t* chunk_dep, int32_t* row_src, mux_pack_info* info,
                        void* workspace, cudaStream_t stream);
cudaError_t launch_pack_apply(int max_rows, int cols, int num_tokens, const int32_t* row_src,
                              const __nv_bfloat16* src, __nv_bfloat16* dst, int num_sms, cudaStream_t stream);
cudaError_t launch_row_start(int num_seqs, const int32_t* seq_len, const int32_t* seq_row, int max_rows,
                             int32_t* row_start, int num_sms, cudaStream_t s);
cudaError_t launch_rmsnorm_fwd(int rows, int dim, const void* x, long long ldx, const void* res, long long ldr,
                               void* xs, long long ldxs, const void* w, float eps, void* y, long long ldy,
                               cudaStream_t s);
cudaError_t launch_rmsnorm_bwd(int rows, int dim, const void* const* dy, const long long* lddy, const void* resid,
                               long long ldr, const void* x, long long ldx, const void* w, float eps, void* dx,
                               long long lddx, cudaStream_t s);
cudaError_t launch_swiglu_fwd(int rows, int dim, const void* g, long long ldg, const void* u, long long ldu, void* h,
                              long long ldh, int num_sms, cudaStream_t s);
cudaError_t launch_swiglu_bwd(int rows, int dim, const void* dh, long long lddh, const void* g, long long ldg,
                              const void* u, long long ldu, void* dg, long long lddg, void* du, long long lddu,
                              int num_sms, cudaStream_t s);
cudaError_t launch_rope(int rows, int heads, int d, void* x, long long ld, const int32_t* row_start, float base,
                        bool inverse, int num_sms, cudaStream_t s);
cudaError_t launch_add(int rows, int dim, const void* a, long long lda, const void* b, long long ldb, void* y,
                       long long ldy, int num_sms, cudaStream_t s);
cudaError_t launch_attn_fwd_tc(const AttnTcParams& p, cudaStream_t s);
cudaError_t launch_rs_reduce(const RsReduceParams& p, int num_sms, cudaStream_t s);
cudaError_t launch_check_segments(int num_segs, const int32_t* seg_off, int max_rows, cudaStream_t s);
cudaError_t launch_attn_bwd_pre(int R, int H, const void* dO, long long lddo, const void* o, long long ldo,
                                float* D, cudaStream_t s);
cudaError_t launch_attn_bwd_tc(const AttnBwdTcParams& p, cudaStream_t s);

}  // namespace mux

using namespace mux;

namespace {

thread_local std::string g_err;

mux_status fail(mux_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

mux_status cuda_fail(cudaError_t e, const char* what) {
  return fail(MUX_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ---- cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// stream memory operations (copy-engine all-gather signalling) through the driver entry points
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
StreamValueFn stream_value_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<StreamValueFn>(p);
  return nullptr;
}
StreamValueFn wait_value64() {
  static StreamValueFn fn = stream_value_fn("cuStreamWaitValue64");
  return fn;
}
StreamValueFn write_value64() {
  static StreamValueFn fn = stream_value_fn("cuStreamWriteValue64");
  return fn;
}

struct MapKey {
  const void* ptr;
  uint64_t inner, outer, stride;
  uint32_t box_inner, box_outer;
  int swizzle;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && stride == o.stride &&
           box_inner == o.box_inner && box_outer == o.box_outer && swizzle == o.swizzle;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.ptr);
    h ^= k.inner * 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h ^= k.outer * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
    h ^= k.stride * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
    h ^= (static_cast<uint64_t>(k.box_inner) << 32 | k.box_outer) + (h << 6) + (h >> 2);
    h ^= static_cast<size_t>(k.swizzle) * 0x9E3779B97F4A7C15ull;
    return h;
  }
};

// A tensor map is a pure function of (address, shape, stride, box): caching
// by that key is exact, and saves the host ~1 us per descriptor per call.
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// 2D bf16 tensor [outer, inner] with row stride `stride` elements, box
// {box_inner, box_outer}, 128 B swizzle (or 32 B: swizzle = 32), zero fill out of bounds.
bool make_map(CUtensorMap* out, const void* ptr, uint64_t inner, uint64_t outer, uint64_t stride,
              uint32_t box_inner, uint32_t box_outer, int swizzle = 128) {
  MapKey key{ptr, inner, outer, stride, box_inner, box_outer, swizzle};
  {
    std::lock_guard<std::mutex> g(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return true;
    }
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  // The driver call needs a current context on this thread.  A thread that has
  // made no runtime call yet (e.g. PyTorch's autograd worker) has none: a
  // no-op runtime call binds the current device's primary context (or keeps
  // the caller's own current context).
  static thread_local bool ctx_bound = false;
  if (!ctx_bound) {
    cudaFree(nullptr);
    ctx_bound = true;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  *out = m;
  std::lock_guard<std::mutex> g(g_map_mu);
  if (g_maps.size() > 16384) g_maps.clear();
  g_maps.emplace(key, m);
  return true;
}

#ifdef MUX_PROFILE
unsigned long long* dbg_counters() {
  static unsigned long long* d = nullptr;
  if (!d) {
    cudaMalloc(&d, 64 * sizeof(unsigned long long));
    cudaMemset(d, 0, 64 * sizeof(unsigned long long));
  }
  return d;
}
#endif

// limit of a device-side wait on another rank (fused AG/RS flags): MUX_PEER_TIMEOUT_S seconds,
// default 600, 0 = wait forever (rank skew is normal; only a protocol bug never completes)
unsigned long long peer_wait_ns() {
  static const unsigned long long ns = [] {
    const char* e = std::getenv("MUX_PEER_TIMEOUT_S");
    double s = 600.0;
    if (e && *e) s = std::atof(e);
    return s <= 0.0 ? 0ull : static_cast<unsigned long long>(s * 1e9);
  }();
  return ns;
}

int num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

// ---- linear-layer workspace: [epoch, done][flags][Gs][Hs scratch][stream-K flags][stream-K partials]
// Zero-filled once by the caller; the GEMM kernel keeps it consistent across launches, so no
// per-call memset: the row-block flags are counters that the last CTA of every launch resets, in a
// region of FIXED size and offset (MUX_MAX_ROWS / 256 entries) — calls with different max_rows or
// r_cap may share the workspace, and the Gs / Hs scratch of one must never land on another's flags
// (it did when the region was sized by max_rows: garbage counters, a watchdog trap).  The stream-K
// flags are epoch-tagged (ptx.cuh flag_arrive), robust to whatever the region held before.
struct LinearWs {
  unsigned long long* epoch;
  unsigned int* done;
  unsigned long long* flags;
  __nv_bfloat16* gs;
  __nv_bfloat16* hs;
  unsigned long long* sk_flags;
  float* sk_part;
  int sk_slots;
  size_t bytes;
};
int num_sms();
LinearWs carve_linear_ws(void* base, int32_t max_rows, int32_t r_cap) {
  LinearWs w{};
  const size_t n_m = (static_cast<size_t>(max_rows) + kPairRows - 1) / kPairRows;
  const size_t h = 256;
  (void)n_m;
  const size_t f = align256(static_cast<size_t>(MUX_MAX_ROWS / kPairRows) * sizeof(unsigned long long));
  const size_t g = align256(static_cast<size_t>(max_rows) * r_cap * 2);
  // one partial 256 x 256 fp32 tile per CTA pair of a full-device launch (stream-K, gemm.cu)
  w.sk_slots = std::min(kSkMaxClusters, num_sms() / 2);
  const size_t skf = align256(static_cast<size_t>(kSkMaxClusters) * sizeof(unsigned long long));
  const size_t skp = static_cast<size_t>(w.sk_slots) * kSkSlotFloats * sizeof(float);
  uint8_t* b = reinterpret_cast<uint8_t*>(base);
  w.epoch = reinterpret_cast<unsigned long long*>(b);
  w.done = reinterpret_cast<unsigned int*>(b ? b + 8 : nullptr);
  w.flags = reinterpret_cast<unsigned long long*>(b ? b + h : nullptr);
  w.gs = reinterpret_cast<__nv_bfloat16*>(b ? b + h + f : nullptr);
  w.hs = reinterpret_cast<__nv_bfloat16*>(b ? b + h + f + g : nullptr);
  w.sk_flags = reinterpret_cast<unsigned long long*>(b ? b + h + f + 2 * g : nullptr);
  w.sk_part = reinterpret_cast<float*>(b ? b + h + f + 2 * g + skf : nullptr);
  w.bytes = h + f + 2 * g + skf + skp;
  return w;
}

// Column slices of the call (NULL = one slice over all N columns), validated.
struct SliceTab {
  int n;
  int off[MUX_MAX_SLICES + 1];
};

mux_status make_slices(const mux_slices* sl, int32_t N, SliceTab* out) {
  if (!sl) {
    out->n = 1;
    out->off[0] = 0;
    out->off[1] = N;
    return MUX_OK;
  }
  if (sl->num_slices < 1 || sl->num_slices > MUX_MAX_SLICES)
    return fail(MUX_ERR_INVALID_ARGUMENT, "num_slices=%d outside [1,%d]", sl->num_slices, MUX_MAX_SLICES);
  out->n = sl->num_slices;
  for (int s = 0; s <= out->n; ++s) out->off[s] = sl->col_off[s];
  if (out->off[0] != 0 || out->off[out->n] != N)
    return fail(MUX_ERR_INVALID_ARGUMENT, "col_off must start at 0 and end at N=%d (got %d .. %d)", N, out->off[0],
                out->off[out->n]);
  for (int s = 0; s < out->n; ++s)
    if (out->off[s + 1] <= out->off[s] || (out->off[s] % 8))
      return fail(MUX_ERR_INVALID_ARGUMENT, "col_off[%d..%d] = %d, %d: slices must be non-empty and start at "
                  "multiples of 8", s, s + 1, out->off[s], out->off[s + 1]);
  return MUX_OK;
}

mux_status validate_linear(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                           int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K,
                           int32_t N, int32_t r_cap, const SliceTab& sl) {
  if (num_segs < 1 || num_segs > MUX_MAX_SEGMENTS)
    return fail(MUX_ERR_INVALID_ARGUMENT, "num_segs=%d outside [1,%d]", num_segs, MUX_MAX_SEGMENTS);
  if (num_adapters < 1 || num_adapters > MUX_MAX_ADAPTERS)
    return fail(MUX_ERR_INVALID_ARGUMENT, "num_adapters=%d outside [1,%d]", num_adapters, MUX_MAX_ADAPTERS);
  if (num_adapters * sl.n > MUX_MAX_ADAPTER_SLOTS)
    return fail(MUX_ERR_INVALID_ARGUMENT, "num_adapters * num_slices = %d * %d > %d adapter slots", num_adapters,
                sl.n, MUX_MAX_ADAPTER_SLOTS);
  if (!seg_off || !seg_task || !adapters) return fail(MUX_ERR_INVALID_ARGUMENT, "null seg_off/seg_task/adapters");
  if (max_rows < 1 || max_rows > MUX_MAX_ROWS)
    return fail(MUX_ERR_INVALID_ARGUMENT, "max_rows=%d outside [1, %d]", max_rows, MUX_MAX_ROWS);
  // multiples of 8: 16-byte TMA row strides; partial 64-wide tiles are handled
  // by TMA zero fill (loads) and clipping (stores)
  if (K < 8 || N < 8 || (K % 8) || (N % 8))
    return fail(MUX_ERR_INVALID_ARGUMENT, "K=%d, N=%d must be positive multiples of 8", K, N);
  if (r_cap != 16 && r_cap != 32 && r_cap != 48 && r_cap != 64)
    return fail(MUX_ERR_INVALID_ARGUMENT, "r_cap=%d must be one of 16, 32, 48, 64", r_cap);
  for (int s = 0; s < num_segs; ++s)
    if (seg_task[s] < 0 || seg_task[s] >= num_adapters)
      return fail(MUX_ERR_INVALID_ARGUMENT, "seg_task[%d]=%d outside [0,%d)", s, seg_task[s], num_adapters);
  for (int t = 0; t < num_adapters * sl.n; ++t) {
    const mux_adapter& a = adapters[t];
    if (a.rank < 0 || a.rank > MUX_MAX_RANK)
      return fail(MUX_ERR_INVALID_ARGUMENT, "adapter %d: rank=%d outside [0,64]", t, a.rank);
    if (a.rank > r_cap) return fail(MUX_ERR_INVALID_ARGUMENT, "adapter %d: rank=%d > r_cap=%d", t, a.rank, r_cap);
    if (!std::isfinite(a.scale)) return fail(MUX_ERR_INVALID_ARGUMENT, "adapter %d: scale is not finite", t);
    if (a.rank > 0) {
      if (!a.A || !a.B) return fail(MUX_ERR_INVALID_ARGUMENT, "adapter %d: null A or B", t);
      if (!aligned16(a.A) || !aligned16(a.B))
        return fail(MUX_ERR_INVALID_ARGUMENT, "adapter %d: A/B not 16-byte aligned", t);
      const int ldb = a.ldb == 0 ? a.rank : a.ldb;
      if (ldb < a.rank || (ldb % 8) != 0)
        return fail(MUX_ERR_INVALID_ARGUMENT,
                    "adapter %d: ldb=%d must be >= rank=%d and a multiple of 8 (16-byte rows for TMA)", t, ldb,
                    a.rank);
    }
  }
  return MUX_OK;
}

// Fill the per-slot TMA descriptors (slot = task * S + slice; B_{t,s} spans the slice's columns).
// A rank-0 slot of a task that has an adapter on another slice gets that slot's descriptors: the
// kernel reads them only at row 64 (all zero fill), so the shrink unit stays uniform.
mux_status fill_adapter_maps(GemmParams& p, int32_t num_adapters, const mux_adapter* adapters, int32_t K,
                             const SliceTab& sl) {
  const int S = sl.n;
  for (int t = 0; t < num_adapters; ++t) {
    int live = -1;
    for (int s = 0; s < S; ++s) {
      const int slot = t * S + s;
      const mux_adapter& a = adapters[slot];
      if (a.rank == 0) continue;
      const int ldb = a.ldb == 0 ? a.rank : a.ldb;
      const int ns = sl.off[s + 1] - sl.off[s];
      if (!make_map(&p.map_lora_a[slot], a.A, K, a.rank, K, 64, 64))
        return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for adapter slot %d A", slot);
      if (!make_map(&p.map_lora_b[slot], a.B, a.rank, ns, ldb, 64, 64))
        return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for adapter slot %d B", slot);
      if (live < 0) live = slot;
    }
    if (live < 0) continue;
    for (int s = 0; s < S; ++s) {
      const int slot = t * S + s;
      if (adapters[slot].rank != 0) continue;
      p.map_lora_a[slot] = p.map_lora_a[live];
      p.map_lora_b[slot] = p.map_lora_b[live];
    }
  }
  return MUX_OK;
}

}  // namespace

mux_status mux_set_error(mux_status st, const char* msg) { return fail(st, "%s", msg); }
unsigned long long mux_peer_wait_ns() { return peer_wait_ns(); }

extern "C" {

const char* mux_last_error(void) { return g_err.c_str(); }

const char* mux_version(void) { return "mux 0.1 sm_100a (tcgen05/TMEM/TMA)"; }

int64_t mux_pack_bound_rows(int64_t total_tokens, int32_t num_seqs, int32_t chunk_size_or_max) {
  if (total_tokens < 0 || num_seqs < 0 || chunk_size_or_max < 1) return -1;
  // every sequence in its own pack, rounded up to the chunk: < total + num_seqs * c
  return total_tokens + static_cast<int64_t>(num_seqs) * chunk_size_or_max;
}

size_t mux_pack_workspace_size(int32_t num_tasks, int32_t num_seqs) {
  return pack_workspace_bytes(num_tasks, num_seqs);
}

mux_status mux_pack_chunks(int32_t num_tasks, int32_t num_seqs, const int32_t* task_seq_off,
                           const int32_t* seq_len, const int32_t* pack_capacity, int32_t chunk_size,
                           int32_t chunk_min, int32_t max_rows, int32_t max_chunks, int32_t* seg_off,
                           int32_t* seq_row, int32_t* chunk_task, int32_t* chunk_pack, int32_t* chunk_valid,
                           int32_t* chunk_dep, int32_t* row_src, mux_pack_info* info, void* workspace,
                           size_t workspace_bytes, cudaStream_t stream) {
  if (num_tasks < 1) return fail(MUX_ERR_INVALID_ARGUMENT, "num_tasks=%d must be >= 1", num_tasks);
  if (num_seqs < 0) return fail(MUX_ERR_INVALID_ARGUMENT, "num_seqs=%d must be >= 0", num_seqs);
  if (chunk_min < 64 || (chunk_min & (chunk_min - 1)))
    return fail(MUX_ERR_INVALID_ARGUMENT, "chunk_min=%d must be a power of two >= 64", chunk_min);
  if (chunk_size != 0 && (chunk_size < 64 || (chunk_size & (chunk_size - 1))))
    return fail(MUX_ERR_INVALID_ARGUMENT, "chunk_size=%d must be 0 or a power of two >= 64", chunk_size);
  if (max_rows < 0 || max_chunks < 0) return fail(MUX_ERR_INVALID_ARGUMENT, "negative capacity");
  if (!task_seq_off || (num_seqs > 0 && !seq_len) || !seg_off || !info)
    return fail(MUX_ERR_INVALID_ARGUMENT, "null required pointer");
  if (num_seqs > 0 && (!seq_row || !chunk_task || !chunk_pack || !chunk_valid || !chunk_dep))
    return fail(MUX_ERR_INVALID_ARGUMENT, "null output pointer");
  if (max_rows > 0 && !row_src) return fail(MUX_ERR_INVALID_ARGUMENT, "null row_src");
  const size_t need = pack_workspace_bytes(num_tasks, num_seqs);
  if (!workspace || workspace_bytes < need)
    return fail(MUX_ERR_INSUFFICIENT_BUFFER, "pack workspace %zu < %zu bytes", workspace_bytes, need);
  cudaError_t e = launch_pack(num_tasks, num_seqs, task_seq_off, seq_len, pack_capacity, chunk_size, chunk_min,
                              max_rows, max_chunks, seg_off, seq_row, chunk_task, chunk_pack, chunk_valid,
                              chunk_dep, row_src, info, workspace, stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_pack_chunks launch");
  return MUX_OK;
}

mux_status mux_pack_apply(int32_t max_rows, int32_t cols, int32_t num_tokens, const int32_t* row_src,
                          const mux_bf16* src_, mux_bf16* dst_, cudaStream_t stream) {
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(src_);
  __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(dst_);
  if (max_rows < 0 || cols < 8 || (cols % 8) || num_tokens < 0)
    return fail(MUX_ERR_INVALID_ARGUMENT, "bad shape max_rows=%d cols=%d num_tokens=%d", max_rows, cols,
                num_tokens);
  if (max_rows == 0) return MUX_OK;
  if (!row_src || !dst || (num_tokens > 0 && !src)) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(src) || !aligned16(dst)) return fail(MUX_ERR_INVALID_ARGUMENT, "src/dst not 16-byte aligned");
  cudaError_t e = launch_pack_apply(max_rows, cols, num_tokens, row_src, src, dst, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_pack_apply launch");
  return MUX_OK;
}

size_t mux_linear_workspace_size(int32_t num_segs, int32_t max_rows, int32_t K, int32_t N, int32_t r_cap) {
  (void)num_segs;
  (void)K;
  (void)N;
  if (max_rows < 0 || r_cap < 0) return 0;
  return carve_linear_ws(nullptr, max_rows, r_cap).bytes;
}

static mux_status linear_common(bool bwd, int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                                int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K,
                                int32_t N, int32_t r_cap, const __nv_bfloat16* a_in /*X or dY*/,
                                const __nv_bfloat16* X, const __nv_bfloat16* W, __nv_bfloat16* out /*Y or dX*/,
                                const __nv_bfloat16* Hs_in, __nv_bfloat16* Hs_out, void* workspace,
                                size_t workspace_bytes, cudaStream_t stream, int parts = 3,
                                const mux_rs* rs = nullptr, const mux_ag* ag = nullptr, bool hs_given = false,
                                bool shrink_only = false, int32_t side_row_lo = 0,
                                int32_t side_row_hi = INT32_MAX, const mux_slices* slices = nullptr,
                                __nv_bfloat16* Gs_ext = nullptr) {
  // Gs_ext (backward only): the caller's Gs [max_rows, S * r_cap] instead of the workspace's — the
  // output of a shrink-only launch, otherwise an input (no shrink tiles; e.g. the rows of a
  // row-parallel layer's Gs computed once per rank and all-gathered, tp.py shared_shrink)
  const bool gs_given = bwd && Gs_ext != nullptr && !shrink_only;
  SliceTab sl;
  mux_status st = make_slices(slices, N, &sl);
  if (st != MUX_OK) return st;
  st = validate_linear(num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap, sl);
  if (st != MUX_OK) return st;
  const int S = sl.n;
  const int side_ld = S * r_cap;  // Hs / Gs row length: slice s at columns [s * r_cap, (s + 1) * r_cap)
  if (!a_in || (!W && !shrink_only)) return fail(MUX_ERR_INVALID_ARGUMENT, "null input pointer");
  if (hs_given && !Hs_in) return fail(MUX_ERR_INVALID_ARGUMENT, "Hs (input) is null");
  if (shrink_only && !(bwd ? Gs_ext : Hs_out))
    return fail(MUX_ERR_INVALID_ARGUMENT, "%s (output) is null", bwd ? "Gs" : "Hs");
  if (shrink_only && (side_row_lo < 0 || side_row_lo % kPairRows || side_row_hi < side_row_lo ||
                      (side_row_hi % kPairRows && side_row_hi < max_rows)))
    return fail(MUX_ERR_INVALID_ARGUMENT, "row range [%d, %d): begin a multiple of 256, end a multiple of 256 or "
                ">= max_rows (%d)", side_row_lo, side_row_hi, max_rows);
  if (!aligned16(a_in) || (W && !aligned16(W)) || (out && !aligned16(out)) || (X && !aligned16(X)) ||
      (Hs_in && !aligned16(Hs_in)) || (Hs_out && !aligned16(Hs_out)) || (Gs_ext && !aligned16(Gs_ext)))
    return fail(MUX_ERR_INVALID_ARGUMENT, "tensor pointers must be 16-byte aligned");
  if (bwd && !shrink_only && (!X || !Hs_in)) return fail(MUX_ERR_INVALID_ARGUMENT, "bwd needs X and Hs");
  if (!bwd && !out && !rs && !shrink_only) return fail(MUX_ERR_INVALID_ARGUMENT, "fwd needs Y");
  const LinearWs need = carve_linear_ws(nullptr, max_rows, side_ld);
  if (!workspace || workspace_bytes < need.bytes)
    return fail(MUX_ERR_INSUFFICIENT_BUFFER, "linear workspace %zu < %zu bytes", workspace_bytes, need.bytes);
  if (!aligned16(workspace)) return fail(MUX_ERR_INVALID_ARGUMENT, "workspace not 16-byte aligned");
  const LinearWs ws = carve_linear_ws(workspace, max_rows, side_ld);

  static thread_local GemmParams p;  // ~17 KB: keep it off the stack
  std::memset(&p, 0, sizeof(p));
  const int kred = bwd ? N : K;
  const int nout = bwd ? K : N;
  __nv_bfloat16* side = bwd ? (Gs_ext ? Gs_ext : ws.gs)
                            : hs_given ? const_cast<__nv_bfloat16*>(Hs_in) : (Hs_out ? Hs_out : ws.hs);
  if (!make_map(&p.map_a, a_in, kred, max_rows, kred, 64, 128))
    return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for %s %p [%d x %d]", bwd ? "dY" : "X", a_in, max_rows, kred);
  if (W && !make_map(&p.map_w, W, K, N, K, 64, 64))
    return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for W %p [%d x %d]", W, N, K);
  if (!make_map(&p.map_side, side, side_ld, max_rows, side_ld, 64, 128))
    return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for %s %p [%d x %d]", bwd ? "Gs" : "Hs", side, max_rows,
                side_ld);
  if (out && !make_map(&p.map_out, out, nout, max_rows, nout, 64, 32))
    return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for %s %p [%d x %d]", bwd ? "dX" : "Y", out, max_rows,
                nout);
  st = fill_adapter_maps(p, num_adapters, adapters, K, sl);
  if (st != MUX_OK) return st;
  p.seg_off = seg_off;
  p.side_out = side;
  p.out = out;
#ifdef MUX_PROFILE
  p.dbg = dbg_counters();
#endif
  p.flags = ws.flags;
  p.epoch = ws.epoch;
  p.done = ws.done;
  p.num_segs = num_segs;
  p.max_rows = max_rows;
  p.kred = kred;
  p.nout = nout;
  p.r_cap = r_cap;
  p.num_slices = S;
  for (int s = 0; s <= S; ++s) p.slice_off[s] = sl.off[s];
  p.has_main = out != nullptr || rs != nullptr;
  p.has_side = (hs_given || gs_given) ? 0 : 1;
  // short reductions: side tiles first (A/B in DESIGN §12: +3-9 % at kred <= 1376, neutral at 4096+)
  p.side_first = kred <= MUX_SIDE_FIRST_MAX_KRED ? 1 : 0;
  p.side_m_lo = side_row_lo / kPairRows;
  p.side_m_hi = side_row_hi == INT32_MAX ? INT32_MAX : (side_row_hi + kPairRows - 1) / kPairRows;
  if (ag) {
    if (ag->world < 1 || ag->world > MUX_RS_MAX_WORLD || ag->rank < 0 || ag->rank >= ag->world || ag->seq == 0 ||
        ag->rows_per_rank <= 0 || ag->rows_per_rank % kPairRows ||
        static_cast<long long>(ag->rows_per_rank) * ag->world != max_rows || !ag->flags[ag->rank])
      return fail(MUX_ERR_INVALID_ARGUMENT, "ag: world=%d rank=%d rows_per_rank=%d (multiple of 256, world * it == "
                  "max_rows=%d), seq > 0, flags", ag->world, ag->rank, ag->rows_per_rank, max_rows);
    p.ag_world = ag->world;
    p.ag_rows = ag->rows_per_rank;
    p.ag_seq = ag->seq;
    p.ag_flags = ag->flags[ag->rank];
  }
  p.peer_wait_ns = peer_wait_ns();
  if (rs) {
    if (rs->world < 1 || rs->world > MUX_RS_MAX_WORLD || rs->rank < 0 || rs->rank >= rs->world)
      return fail(MUX_ERR_INVALID_ARGUMENT, "rs: world=%d rank=%d", rs->world, rs->rank);
    if (rs->rows_per_rank <= 0 || rs->rows_per_rank % kPairRows ||
        static_cast<long long>(rs->rows_per_rank) * rs->world != max_rows)
      return fail(MUX_ERR_INVALID_ARGUMENT, "rs: rows_per_rank=%d must be a multiple of 256 with world * it == "
                  "max_rows=%d", rs->rows_per_rank, max_rows);
    if (rs->seq == 0) return fail(MUX_ERR_INVALID_ARGUMENT, "rs: seq must be > 0");
    for (int d = 0; d < rs->world; ++d) {
      if (!rs->recv[d] || !rs->flags[d] || !aligned16(rs->recv[d]))
        return fail(MUX_ERR_INVALID_ARGUMENT, "rs: recv/flags of rank %d null or misaligned", d);
      const __nv_bfloat16* slot = reinterpret_cast<const __nv_bfloat16*>(rs->recv[d]) +
                                  static_cast<size_t>(rs->rank) * rs->rows_per_rank * nout;
      if (!make_map(&p.map_out_rs[d], slot, nout, rs->rows_per_rank, nout, 64, 32))
        return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for the receive slot on rank %d", d);
      p.rs_ready[d] = rs->flags[d] + rs->rank;
    }
    p.rs_world = rs->world;
    p.rs_rows = rs->rows_per_rank;
    p.rs_seq = rs->seq;
    p.rs_ack = rs->flags[rs->rank] + rs->world;
  }
  // raster band: keep the band's A rows (group_m * 256 rows * kred * 2 B)
  // within ~48 MB of the 126 MB L2, leaving room for the streamed W tiles
#ifndef MUX_GRAD_SIMT_MAX_RANK
#define MUX_GRAD_SIMT_MAX_RANK 0
#endif
#ifndef MUX_BAND_MB
#define MUX_BAND_MB 48
#endif
#ifndef MUX_BAND_MIN
#define MUX_BAND_MIN 4
#endif
#ifndef MUX_RASTER_DEFAULT
#define MUX_RASTER_DEFAULT 'm'   // 'a' = traffic model, 'm' = row bands, 'n' = column bands
#endif
  {
    const long long band_bytes = static_cast<long long>(kPairRows) * kred * 2;
    long long g = (static_cast<long long>(MUX_BAND_MB) << 20) / band_bytes;
    p.group_m = static_cast<int32_t>(std::max(static_cast<long long>(MUX_BAND_MIN), std::min(32ll, g)));
  }
  // raster direction by a DRAM-traffic model: row bands read A once and W once per band; column
  // bands (the band's W tiles L2-resident) read W once and A once per band.  Column bands where
  // they move at most 80 % of the bytes (long reductions with W the smaller operand, e.g. the
  // 11008 -> 4096 down projection); MUX_RASTER=m / n forces one (A/B; read per call).
  {
    const char* re = std::getenv("MUX_RASTER");
    const char rc = (re && *re) ? re[0] : MUX_RASTER_DEFAULT;
    const long long nrow_blk = (static_cast<long long>(max_rows) + kPairRows - 1) / kPairRows;
    const int tile_n0 = nout <= MUX_NARROW_MAX_NOUT ? kBN / 2 : kBN;
    const long long ncol_blk = (static_cast<long long>(nout) + tile_n0 - 1) / tile_n0;
    const long long col_band_bytes = static_cast<long long>(tile_n0) * kred * 2;
    const long long gn = std::max(static_cast<long long>(MUX_BAND_MIN),
                                  std::min(64ll, (static_cast<long long>(MUX_BAND_MB) << 20) / col_band_bytes));
    const double a_bytes = static_cast<double>(max_rows) * kred * 2, w_bytes = static_cast<double>(nout) * kred * 2;
    const double row_bands = a_bytes + w_bytes * static_cast<double>((nrow_blk + p.group_m - 1) / p.group_m);
    const double col_bands = w_bytes + a_bytes * static_cast<double>((ncol_blk + gn - 1) / gn);
    const bool col = rc == 'n' || (rc != 'm' && col_bands <= 0.8 * row_bands);
    p.group_n = (col && !p.side_first) ? static_cast<int32_t>(gn) : 0;
  }
  for (int t = 0; t < num_adapters * S; ++t) {
    p.slot_rank[t] = adapters[t].rank;
    p.slot_scale[t] = adapters[t].scale;
  }
  for (int s = 0; s < num_segs; ++s) {
    int r = 0;
    for (int c = 0; c < S; ++c) r = std::max(r, adapters[seg_task[s] * S + c].rank);
    p.seg_adapter[s] = seg_task[s];
    p.seg_rank[s] = r;
  }
  const int num_m_max = (max_rows + kPairRows - 1) / kPairRows;
  // narrow outputs (<= MUX_NARROW_MAX_NOUT columns): 256 x 128 tiles, twice as many work items;
  // wide outputs (>= MUX_WIDE_MIN_NOUT): 256 x 512 tiles; MUX_TILE_N=128/256/512 forces one (A/B,
  // read per call)
  int tile_n = nout <= MUX_NARROW_MAX_NOUT ? kBN / 2 : nout >= MUX_WIDE_MIN_NOUT ? 2 * kBN : kBN;
  {
    const char* te = std::getenv("MUX_TILE_N");
    const int tv = (te && *te) ? std::atoi(te) : 0;
    if (tv == 128 || tv == 256 || tv == 512) tile_n = tv;
  }
  const int num_n = (nout + tile_n - 1) / tile_n;
  const long long side_blocks = p.has_main ? (p.has_side ? num_m_max : 0)
                                           : std::max(0, std::min(p.side_m_hi, num_m_max) - std::min(p.side_m_lo, num_m_max));
  const long long tiles_max = side_blocks + (p.has_main ? static_cast<long long>(num_m_max) * num_n : 0);
  // one CTA pair (cluster of 2) per tile in flight; grid = #SMs rounded to pairs
  const long long pairs = std::min<long long>(tiles_max, num_sms() / 2);
  const int grid = static_cast<int>(2 * std::max<long long>(pairs, 1));
  // Stream-K (gemm.cu) is built and parity-tested but OFF by default: interleaved A/B on the
  // tensor-parallel shard shapes it targets (profiles/r02_sk_ab_*.jsonl: 512-column outputs and
  // 512-deep reductions, 21.5k rows, 16 tasks) has it 5-25 % SLOWER than whole tiles, because the
  // kernel is bound by the operand feed, not by idle CTA pairs: a last round with a third of the
  // pairs busy runs those tiles faster, and the split adds partial traffic.  MUX_SK=1 forces it
  // (tests, A/B); MUX_SK=-1 enables the quantization heuristic (balanced load < 0.85 x rounds).
  {
    const char* sk_e = std::getenv("MUX_SK");  // read per call: tests compare both schedules in one process
    const int sk_env = (sk_e && *sk_e) ? std::atoi(sk_e) : 0;
    static const int side_cost_x4 = [] {
      const char* e = std::getenv("MUX_SK_SIDE_COST_X4");
      return (e && *e) ? std::atoi(e) : 3;
    }();
    const int num_kb = (kred + GemmCfg<false>::kBK - 1) / GemmCfg<false>::kBK;
    const long long main_tiles = p.has_main ? static_cast<long long>(num_m_max) * num_n : 0;
    const double ideal = (main_tiles + side_blocks * side_cost_x4 / 4.0) / pairs;
    const double rounds = static_cast<double>((tiles_max + pairs - 1) / pairs);
    const bool fits = p.has_main && pairs <= ws.sk_slots && pairs <= kSkMaxClusters && num_kb >= 2 &&
                      tile_n <= kBN;  // partial slots hold 256-column tiles
    p.sk = fits && (sk_env == 1 || (sk_env < 0 && ideal < 0.85 * rounds)) ? 1 : 0;
    p.sk_side_cost_x4 = side_cost_x4;
    p.sk_flags = ws.sk_flags;
    p.sk_part = ws.sk_part;
  }
  // Carrier shrink (gemm.cu tile_at_carry): the shrink rides on the first main tiles of each row
  // block instead of side tiles, which re-read X / dY and, at config 2, push the tile count just past
  // a wave of CTA pairs (profiles/r02_shrink_cost.jsonl: side tiles 10-12 % of four of the six
  // GEMMs).  Needs one slice, r_cap <= 32 (32 stacked adapter rows per carrier), <= 32 adapters,
  // standard tiles, no stream-K, and enough column tiles for the carriers (<= 4 task groups per row
  // block).  MUX_CARRY=0 keeps the side tiles, 2 forces carriers at short reductions too (A/B; read
  // per call).
  {
#ifndef MUX_CARRY_DEFAULT
#define MUX_CARRY_DEFAULT 1
#endif
    const char* ce = std::getenv("MUX_CARRY");
    const int cv = (ce && *ce) ? std::atoi(ce) : MUX_CARRY_DEFAULT;
    int live = 0;
    for (int i = 0; i < num_segs; ++i) live += p.seg_rank[i] > 0 ? 1 : 0;
    const int gpc = r_cap <= 32 ? 32 / r_cap : 1;
    const int nc_max = std::max(1, (std::min(4, live) + gpc - 1) / gpc);
    // Short reductions (<= MUX_SIDE_FIRST_MAX_KRED) keep the side tiles, all first: there a
    // carrier's own shrink round trip (epilogue -> Hs -> flag -> extension block) is as long as a
    // whole tile (profiles/r02_carry1_ab_tp_fwd.jsonl: 512 -> 4096 +13 %).  The kernel itself falls
    // back to side tiles when the carriers would not fit one wave of CTA pairs.
    if (cv != 0 && p.has_main && p.has_side && S == 1 && r_cap <= 32 && tile_n == kBN && !p.sk &&
        nc_max <= num_n && num_adapters <= kMaxCarrySlots && (cv >= 2 || kred > MUX_SIDE_FIRST_MAX_KRED)) {
      // MUX_CARRY=3: also when one carrier per row block spans more than one wave (A/B)
      p.carry = cv == 3 ? 2 : 1;
      for (int t = 0; t < num_adapters; ++t) {
        const mux_adapter& a = adapters[t];
        if (a.rank == 0) continue;
        const int ldb = a.ldb == 0 ? a.rank : a.ldb;
        const bool ok = bwd ? make_map(&p.map_shrink[t], a.B, a.rank, N, ldb, 16, 128, 32)  // B_t MN-major
                            : make_map(&p.map_shrink[t], a.A, K, a.rank, K, 64, 8);        // A_t K-major
        if (!ok) return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for the shrink map of adapter %d", t);
      }
    }
  }
  cudaError_t e = cudaSuccess;
#ifdef MUX_DEBUG_CHECKS
  e = launch_check_segments(num_segs, seg_off, max_rows, stream);
  if (e != cudaSuccess) return cuda_fail(e, "debug segment check launch");
#endif
  if (parts & 1) {
    e = launch_gemm(p, bwd, tile_n, grid, stream);
    if (e != cudaSuccess) return cuda_fail(e, bwd ? "mux_linear_bwd dX launch" : "mux_linear_fwd launch");
  }

  int grad_max_rank = 0;
  for (int i = 0; i < num_adapters * S; ++i)
    if (adapters[i].dA || adapters[i].dB) grad_max_rank = std::max(grad_max_rank, adapters[i].rank);
  if (bwd && (parts & 2) && grad_max_rank > MUX_GRAD_SIMT_MAX_RANK) {
    // tensor cores (grad.cu): every slice in one launch; X is streamed once for all slices' dA
    static thread_local GradParams g;
    std::memset(&g, 0, sizeof(g));
    __nv_bfloat16* gs_src = Gs_ext ? Gs_ext : ws.gs;
    if (!make_map(&g.map_x, X, K, max_rows, K, 64, 128) || !make_map(&g.map_dy, a_in, N, max_rows, N, 64, 128) ||
        !make_map(&g.map_hs, Hs_in, S * r_cap, max_rows, side_ld, 64, 128) ||
        !make_map(&g.map_gs, gs_src, S * r_cap, max_rows, side_ld, 64, 128))
      return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for a gradient-kernel operand (X, dY, Hs or Gs)");
    g.seg_off = seg_off;
    g.num_segs = num_segs;
    g.K = K;
    g.N = N;
    g.r_cap = r_cap;
    g.num_slices = S;
    bool want_a = false, want_b = false;
    int nt = 0;
    for (int t = 0; t < num_adapters; ++t) {
      bool live = false;
      for (int sc = 0; sc < S; ++sc) {
        const mux_adapter& a = adapters[t * S + sc];
        live |= a.rank > 0 && (a.dA || a.dB);
      }
      if (!live) continue;
      uint64_t segs = 0;
      for (int s = 0; s < num_segs; ++s)
        if (seg_task[s] == t) segs |= 1ull << s;
      g.task_segs[nt] = segs;
      for (int sc = 0; sc < S; ++sc) {
        const mux_adapter& a = adapters[t * S + sc];
        g.slot_rank[nt * S + sc] = a.rank;
        g.slot_dA[nt * S + sc] = a.rank > 0 ? a.dA : nullptr;
        g.slot_dB[nt * S + sc] = a.rank > 0 ? a.dB : nullptr;
        want_a |= a.rank > 0 && a.dA != nullptr;
        want_b |= a.rank > 0 && a.dB != nullptr;
      }
      ++nt;
    }
    g.num_tasks = nt;
    g.nb_a = (S * r_cap + 63) / 64;
    g.units_a = want_a ? (K + kGradBM - 1) / kGradBM : 0;
    g.slice_off[0] = 0;
    g.b_units_off[0] = 0;
    for (int sc = 0; sc < S; ++sc) {
      g.slice_off[sc + 1] = sl.off[sc + 1];
      const int n_s = sl.off[sc + 1] - sl.off[sc];
      g.b_units_off[sc + 1] = g.b_units_off[sc] + (want_b ? (n_s + kGradBM - 1) / kGradBM : 0);
    }
    for (int sc = S + 1; sc <= MUX_MAX_SLICES; ++sc) g.slice_off[sc] = g.b_units_off[sc] = 0;
    g.units_b = g.b_units_off[S];
    // stage = 128 rows of X / dY (32 KB) + the B boxes (16 KB each): 4 stages of 48 KB down to 2 of 96 KB
    g.stage_bytes = 2u * kGradBK * 128u + static_cast<uint32_t>(std::max(g.nb_a, 1)) * kGradBK * 128u;
    g.stages = std::min<int>(kGradStages, (kGradStages * 3u * kGradBK * 128u) / g.stage_bytes);
    const long long units = static_cast<long long>(nt) * (g.units_a + g.units_b);
    if (units > 0) {
      // HBM-bound: spread the units evenly (every CTA gets the same number of units) instead of
      // leaving a ragged last wave on 148 CTAs
      const long long waves = (units + num_sms() - 1) / num_sms();
      const int ggrid = static_cast<int>((units + waves - 1) / waves);
      e = launch_grad(g, ggrid, stream);
      if (e != cudaSuccess) return cuda_fail(e, "mux_linear_bwd grad launch");
    }
  } else if (bwd && (parts & 2)) {
    // CUDA-core kernel (grad_simt.cu, MUX_GRAD_SIMT_MAX_RANK builds): one launch per column slice s:
    // dY's columns of the slice, Hs_s / Gs_s (columns [s * r_cap, (s + 1) * r_cap) of the side
    // tensors), the slots (t, s)
    for (int sc = 0; sc < S; ++sc) {
      static thread_local GradParams g;
      std::memset(&g, 0, sizeof(g));
      const int n_s = sl.off[sc + 1] - sl.off[sc];
      if (!make_map(&g.map_x, X, K, max_rows, K, 64, 128) ||
          !make_map(&g.map_dy, a_in + sl.off[sc], n_s, max_rows, N, 64, 128) ||
          !make_map(&g.map_hs, Hs_in + sc * r_cap, r_cap, max_rows, side_ld, 64, 128) ||
          !make_map(&g.map_gs, (Gs_ext ? Gs_ext : ws.gs) + sc * r_cap, r_cap, max_rows, side_ld, 64, 128))
        return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for a gradient-kernel operand (X, dY, Hs or Gs)");
      g.seg_off = seg_off;
      g.num_segs = num_segs;
      g.K = K;
      g.N = n_s;
      g.r_cap = r_cap;
      bool want_a = false, want_b = false;
      int nt = 0;
      int max_rank = 0;
      for (int t = 0; t < num_adapters; ++t) {
        const mux_adapter& a = adapters[t * S + sc];
        if (a.rank == 0 || (!a.dA && !a.dB)) continue;
        uint64_t segs = 0;
        for (int s = 0; s < num_segs; ++s)
          if (seg_task[s] == t) segs |= 1ull << s;
        g.task_segs[nt] = segs;
        g.task_rank[nt] = a.rank;
        g.task_dA[nt] = a.dA;
        g.task_dB[nt] = a.dB;
        want_a |= a.dA != nullptr;
        want_b |= a.dB != nullptr;
        max_rank = std::max(max_rank, a.rank);
        ++nt;
      }
      g.num_tasks = nt;
      g.units_a = want_a ? (K + kGradBM - 1) / kGradBM : 0;
      g.units_b = want_b ? (n_s + kGradBM - 1) / kGradBM : 0;
      const long long units = static_cast<long long>(nt) * (g.units_a + g.units_b);
      if (units > 0) {
        // HBM-bound: spread the units evenly (every CTA gets the same number of
        // units) instead of leaving a ragged last wave on 148 CTAs
        const long long waves = (units + num_sms() - 1) / num_sms();
        const int ggrid = static_cast<int>((units + waves - 1) / waves);
        // every rank is at most MUX_GRAD_SIMT_MAX_RANK (0 by default: DESIGN §6.2's A/B)
        (void)max_rank;
        e = launch_grad_simt(g, ggrid, stream);
        if (e != cudaSuccess) return cuda_fail(e, "mux_linear_bwd grad launch");
      }
    }
  }
  return MUX_OK;
}

mux_status mux_linear_fwd(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                          int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K, int32_t N,
                          int32_t r_cap, const mux_bf16* X_, const mux_bf16* W_, mux_bf16* Y_,
                          mux_bf16* Hs_, void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  auto X = reinterpret_cast<const __nv_bfloat16*>(X_);
  auto W = reinterpret_cast<const __nv_bfloat16*>(W_);
  auto Y = reinterpret_cast<__nv_bfloat16*>(Y_);
  auto Hs = reinterpret_cast<__nv_bfloat16*>(Hs_);
  return linear_common(false, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap, X, X, W,
                       Y, nullptr, Hs, workspace, workspace_bytes, stream);
}

mux_status mux_linear_fwd_hs(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                             int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K, int32_t N,
                             int32_t r_cap, const mux_bf16* X_, const mux_bf16* W_, mux_bf16* Y_,
                             const mux_bf16* Hs_, void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  auto X = reinterpret_cast<const __nv_bfloat16*>(X_);
  return linear_common(false, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap, X, X,
                       reinterpret_cast<const __nv_bfloat16*>(W_), reinterpret_cast<__nv_bfloat16*>(Y_),
                       reinterpret_cast<const __nv_bfloat16*>(Hs_), nullptr, workspace, workspace_bytes, stream, 3,
                       nullptr, nullptr, /*hs_given=*/true);
}

mux_status mux_linear_shrink(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                             int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K, int32_t N,
                             int32_t r_cap, const mux_bf16* X_, int32_t row_begin, int32_t row_end, mux_bf16* Hs_,
                             void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  auto X = reinterpret_cast<const __nv_bfloat16*>(X_);
  return linear_common(false, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap, X, X,
                       nullptr, nullptr, nullptr, reinterpret_cast<__nv_bfloat16*>(Hs_), workspace, workspace_bytes,
                       stream, 3, nullptr, nullptr, false, /*shrink_only=*/true, row_begin, row_end);
}

mux_status mux_linear_bwd(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                          int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K, int32_t N,
                          int32_t r_cap, const mux_bf16* dY_, const mux_bf16* X_, const mux_bf16* W_,
                          const mux_bf16* Hs_, mux_bf16* dX_, void* workspace, size_t workspace_bytes,
                          cudaStream_t stream) {
  auto dY = reinterpret_cast<const __nv_bfloat16*>(dY_);
  auto X = reinterpret_cast<const __nv_bfloat16*>(X_);
  auto W = reinterpret_cast<const __nv_bfloat16*>(W_);
  auto Hs = reinterpret_cast<const __nv_bfloat16*>(Hs_);
  auto dX = reinterpret_cast<__nv_bfloat16*>(dX_);
  return linear_common(true, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap, dY, X, W,
                       dX, Hs, nullptr, workspace, workspace_bytes, stream);
}

mux_status mux_linear_bwd_part(int32_t part, int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                               int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K,
                               int32_t N, int32_t r_cap, const mux_bf16* dY_, const mux_bf16* X_, const mux_bf16* W_,
                               const mux_bf16* Hs_, mux_bf16* dX_, void* workspace, size_t workspace_bytes,
                               cudaStream_t stream) {
  if (part != MUX_BWD_DX && part != MUX_BWD_GRADS)
    return fail(MUX_ERR_INVALID_ARGUMENT, "part=%d must be MUX_BWD_DX (1) or MUX_BWD_GRADS (2)", part);
  return linear_common(true, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap,
                       reinterpret_cast<const __nv_bfloat16*>(dY_), reinterpret_cast<const __nv_bfloat16*>(X_),
                       reinterpret_cast<const __nv_bfloat16*>(W_), reinterpret_cast<__nv_bfloat16*>(dX_),
                       reinterpret_cast<const __nv_bfloat16*>(Hs_), nullptr, workspace, workspace_bytes, stream,
                       part);
}

#ifdef MUX_PROFILE
// [host] experiment builds only: synchronizes, copies and resets the wait-cycle counters.
MUX_API int mux_debug_counters(unsigned long long* host_out, int n) {
  unsigned long long* d = dbg_counters();
  cudaDeviceSynchronize();
  cudaMemcpy(host_out, d, sizeof(unsigned long long) * (n < 64 ? n : 64), cudaMemcpyDeviceToHost);
  cudaMemset(d, 0, 64 * sizeof(unsigned long long));
  return 0;
}
#endif


// ---------------------------------------------------------------- decoder-block ops (NEXT-3)
static bool ld_ok(long long ld, int cols) { return ld >= cols && ld % 8 == 0; }

mux_status mux_pack_row_start(int32_t num_seqs, const int32_t* seq_len, const int32_t* seq_row, int32_t max_rows,
                              int32_t* row_start, cudaStream_t stream) {
  if (num_seqs < 0 || max_rows < 0)
    return fail(MUX_ERR_INVALID_ARGUMENT, "bad sizes num_seqs=%d max_rows=%d", num_seqs, max_rows);
  if (max_rows == 0) return MUX_OK;
  if (!row_start || (num_seqs > 0 && (!seq_len || !seq_row))) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  cudaError_t e = launch_row_start(num_seqs, seq_len, seq_row, max_rows, row_start, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_pack_row_start launch");
  return MUX_OK;
}

static mux_status attn_check(int32_t rows, int32_t heads, int32_t kv_heads, int32_t head_dim) {
  if (rows < 0 || heads < 1 || kv_heads < 1 || heads % kv_heads)
    return fail(MUX_ERR_INVALID_ARGUMENT, "bad attention sizes rows=%d heads=%d kv_heads=%d", rows, heads, kv_heads);
  if (head_dim != 128) return fail(MUX_ERR_UNSUPPORTED, "head_dim=%d (this build: 128)", head_dim);
  return MUX_OK;
}

mux_status mux_attn_fwd(int32_t rows, int32_t heads, int32_t kv_heads, int32_t head_dim, const mux_bf16* q,
                        int64_t ldq, const mux_bf16* k, int64_t ldk, const mux_bf16* v, int64_t ldv,
                        const int32_t* row_start, float scale, mux_bf16* o, int64_t ldo, float* lse,
                        cudaStream_t stream) {
  mux_status st = attn_check(rows, heads, kv_heads, head_dim);
  if (st != MUX_OK || rows == 0) return st;
  if (!q || !k || !v || !row_start || !o || !lse) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(MUX_ERR_INVALID_ARGUMENT, "q/k/v/o not 16-byte aligned");
  if (!ld_ok(ldq, heads * 128) || !ld_ok(ldo, heads * 128) || !ld_ok(ldk, kv_heads * 128) ||
      !ld_ok(ldv, kv_heads * 128))
    return fail(MUX_ERR_INVALID_ARGUMENT, "row strides must cover the heads and be multiples of 8");
  if (!std::isfinite(scale)) return fail(MUX_ERR_INVALID_ARGUMENT, "scale not finite");
  static thread_local AttnTcParams ap;
  if (!make_map(&ap.map_q, q, heads * 128, rows, ldq, 64, 128) ||
      !make_map(&ap.map_k, k, kv_heads * 128, rows, ldk, 64, 64) ||
      !make_map(&ap.map_v, v, kv_heads * 128, rows, ldv, 64, 64))
    return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for q/k/v");
  ap.row_start = row_start;
  ap.o = reinterpret_cast<__nv_bfloat16*>(o);
  ap.ldo = ldo;
  ap.lse = lse;
  ap.R = rows;
  ap.H = heads;
  ap.Hkv = kv_heads;
  ap.scale_log2 = scale * 1.4426950408889634f;
  cudaError_t e = launch_attn_fwd_tc(ap, stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_attn_fwd launch");
  return MUX_OK;
}

size_t mux_attn_workspace_size(int32_t rows, int32_t heads) {
  if (rows < 0 || heads < 0) return 0;
  return align256(sizeof(float) * static_cast<size_t>(rows) * heads);
}

mux_status mux_attn_bwd(int32_t rows, int32_t heads, int32_t kv_heads, int32_t head_dim, const mux_bf16* dO,
                        int64_t lddo, const mux_bf16* q, int64_t ldq, const mux_bf16* k, int64_t ldk,
                        const mux_bf16* v, int64_t ldv, const mux_bf16* o, int64_t ldo, const float* lse,
                        const int32_t* row_start, float scale, mux_bf16* dq, int64_t lddq, mux_bf16* dk,
                        int64_t lddk, mux_bf16* dv, int64_t lddv, void* workspace, size_t workspace_bytes,
                        cudaStream_t stream) {
  mux_status st = attn_check(rows, heads, kv_heads, head_dim);
  if (st != MUX_OK || rows == 0) return st;
  if (!dO || !q || !k || !v || !o || !lse || !row_start || !dq || !dk || !dv)
    return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(dO) || !aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(dq) ||
      !aligned16(dk) || !aligned16(dv))
    return fail(MUX_ERR_INVALID_ARGUMENT, "tensors must be 16-byte aligned");
  const int qc = heads * 128, kc = kv_heads * 128;
  if (!ld_ok(lddo, qc) || !ld_ok(ldq, qc) || !ld_ok(ldo, qc) || !ld_ok(lddq, qc) || !ld_ok(ldk, kc) ||
      !ld_ok(ldv, kc) || !ld_ok(lddk, kc) || !ld_ok(lddv, kc))
    return fail(MUX_ERR_INVALID_ARGUMENT, "row strides must cover the heads and be multiples of 8");
  if (!std::isfinite(scale)) return fail(MUX_ERR_INVALID_ARGUMENT, "scale not finite");
  const size_t need = mux_attn_workspace_size(rows, heads);
  if (!workspace || workspace_bytes < need)
    return fail(MUX_ERR_INSUFFICIENT_BUFFER, "attention workspace %zu < %zu bytes", workspace_bytes, need);
  static thread_local AttnBwdTcParams bp;
  const int qc2 = heads * 128, kc2 = kv_heads * 128;
  if (!make_map(&bp.map_q128, q, qc2, rows, ldq, 64, 128) || !make_map(&bp.map_do128, dO, qc2, rows, lddo, 64, 128) ||
      !make_map(&bp.map_q64, q, qc2, rows, ldq, 64, 64) || !make_map(&bp.map_do64, dO, qc2, rows, lddo, 64, 64) ||
      !make_map(&bp.map_k64, k, kc2, rows, ldk, 64, 64) || !make_map(&bp.map_v64, v, kc2, rows, ldv, 64, 64) ||
      !make_map(&bp.map_k128, k, kc2, rows, ldk, 64, 128) || !make_map(&bp.map_v128, v, kc2, rows, ldv, 64, 128))
    return fail(MUX_ERR_CUDA, "cuTensorMapEncodeTiled failed for q/k/v/dO");
  bp.row_start = row_start;
  bp.lse = lse;
  bp.D = static_cast<const float*>(workspace);
  bp.dq = reinterpret_cast<__nv_bfloat16*>(dq);
  bp.lddq = lddq;
  bp.dk = reinterpret_cast<__nv_bfloat16*>(dk);
  bp.lddk = lddk;
  bp.dv = reinterpret_cast<__nv_bfloat16*>(dv);
  bp.lddv = lddv;
  bp.R = rows;
  bp.H = heads;
  bp.Hkv = kv_heads;
  bp.scale_log2 = scale * 1.4426950408889634f;
  bp.scale = scale;
  cudaError_t e = launch_attn_bwd_pre(rows, heads, dO, lddo, o, ldo, static_cast<float*>(workspace), stream);
  if (e == cudaSuccess) e = launch_attn_bwd_tc(bp, stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_attn_bwd launch");
  return MUX_OK;
}

mux_status mux_rope(int32_t rows, int32_t heads, int32_t head_dim, mux_bf16* x, int64_t ld,
                    const int32_t* row_start, float base, int32_t inverse, cudaStream_t stream) {
  if (rows < 0 || heads < 1 || head_dim < 16 || head_dim % 16)
    return fail(MUX_ERR_INVALID_ARGUMENT, "bad rope sizes rows=%d heads=%d head_dim=%d", rows, heads, head_dim);
  if (rows == 0) return MUX_OK;
  if (!x || !row_start) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(x) || !ld_ok(ld, heads * head_dim)) return fail(MUX_ERR_INVALID_ARGUMENT, "x alignment/stride");
  if (!(base > 1.f) || !std::isfinite(base)) return fail(MUX_ERR_INVALID_ARGUMENT, "rope base must be > 1");
  cudaError_t e = launch_rope(rows, heads, head_dim, x, ld, row_start, base, inverse != 0, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_rope launch");
  return MUX_OK;
}

static mux_status ew_check(int32_t rows, int32_t dim) {
  if (rows < 0 || dim < 8 || dim % 8) return fail(MUX_ERR_INVALID_ARGUMENT, "bad sizes rows=%d dim=%d", rows, dim);
  return MUX_OK;
}

mux_status mux_rmsnorm_fwd(int32_t rows, int32_t dim, const mux_bf16* x, int64_t ldx, const mux_bf16* res,
                           int64_t ldres, mux_bf16* xsum, int64_t ldxs, const mux_bf16* w, float eps, mux_bf16* y,
                           int64_t ldy, cudaStream_t stream) {
  mux_status st = ew_check(rows, dim);
  if (st != MUX_OK || rows == 0) return st;
  if (!x || !w || !y) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(x) || !aligned16(w) || !aligned16(y) || !ld_ok(ldx, dim) || !ld_ok(ldy, dim) ||
      (res && (!aligned16(res) || !ld_ok(ldres, dim))) || (xsum && (!aligned16(xsum) || !ld_ok(ldxs, dim))))
    return fail(MUX_ERR_INVALID_ARGUMENT, "alignment/stride");
  if (xsum && !res) return fail(MUX_ERR_INVALID_ARGUMENT, "xsum needs res");
  if (!(eps >= 0.f) || !std::isfinite(eps)) return fail(MUX_ERR_INVALID_ARGUMENT, "eps must be finite and >= 0");
  cudaError_t e = launch_rmsnorm_fwd(rows, dim, x, ldx, res, ldres, xsum, ldxs, w, eps, y, ldy, stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_rmsnorm_fwd launch");
  return MUX_OK;
}

mux_status mux_rmsnorm_bwd(int32_t rows, int32_t dim, const mux_bf16* dy, int64_t lddy, const mux_bf16* dy2,
                           int64_t lddy2, const mux_bf16* dy3, int64_t lddy3, const mux_bf16* x, int64_t ldx,
                           const mux_bf16* w, float eps, const mux_bf16* resid, int64_t ldres, mux_bf16* dx,
                           int64_t lddx, cudaStream_t stream) {
  mux_status st = ew_check(rows, dim);
  if (st != MUX_OK || rows == 0) return st;
  if (!dy || !x || !w || !dx || (dy3 && !dy2)) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(dy) || !aligned16(x) || !aligned16(w) || !aligned16(dx) || !ld_ok(lddy, dim) || !ld_ok(ldx, dim) ||
      !ld_ok(lddx, dim) || (dy2 && (!aligned16(dy2) || !ld_ok(lddy2, dim))) ||
      (dy3 && (!aligned16(dy3) || !ld_ok(lddy3, dim))) || (resid && (!aligned16(resid) || !ld_ok(ldres, dim))))
    return fail(MUX_ERR_INVALID_ARGUMENT, "alignment/stride");
  if (!(eps >= 0.f) || !std::isfinite(eps)) return fail(MUX_ERR_INVALID_ARGUMENT, "eps must be finite and >= 0");
  const void* dys[3] = {dy, dy2, dy3};
  const long long lds[3] = {lddy, lddy2, lddy3};
  cudaError_t e = launch_rmsnorm_bwd(rows, dim, dys, lds, resid, ldres, x, ldx, w, eps, dx, lddx, stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_rmsnorm_bwd launch");
  return MUX_OK;
}

mux_status mux_swiglu_fwd(int32_t rows, int32_t dim, const mux_bf16* g, int64_t ldg, const mux_bf16* u, int64_t ldu,
                          mux_bf16* h, int64_t ldh, cudaStream_t stream) {
  mux_status st = ew_check(rows, dim);
  if (st != MUX_OK || rows == 0) return st;
  if (!g || !u || !h) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(g) || !aligned16(u) || !aligned16(h) || !ld_ok(ldg, dim) || !ld_ok(ldu, dim) || !ld_ok(ldh, dim))
    return fail(MUX_ERR_INVALID_ARGUMENT, "alignment/stride");
  cudaError_t e = launch_swiglu_fwd(rows, dim, g, ldg, u, ldu, h, ldh, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_swiglu_fwd launch");
  return MUX_OK;
}

mux_status mux_swiglu_bwd(int32_t rows, int32_t dim, const mux_bf16* dh, int64_t lddh, const mux_bf16* g,
                          int64_t ldg, const mux_bf16* u, int64_t ldu, mux_bf16* dg, int64_t lddg, mux_bf16* du,
                          int64_t lddu, cudaStream_t stream) {
  mux_status st = ew_check(rows, dim);
  if (st != MUX_OK || rows == 0) return st;
  if (!dh || !g || !u || !dg || !du) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(dh) || !aligned16(g) || !aligned16(u) || !aligned16(dg) || !aligned16(du) || !ld_ok(lddh, dim) ||
      !ld_ok(ldg, dim) || !ld_ok(ldu, dim) || !ld_ok(lddg, dim) || !ld_ok(lddu, dim))
    return fail(MUX_ERR_INVALID_ARGUMENT, "alignment/stride");
  cudaError_t e = launch_swiglu_bwd(rows, dim, dh, lddh, g, ldg, u, ldu, dg, lddg, du, lddu, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_swiglu_bwd launch");
  return MUX_OK;
}

mux_status mux_add(int32_t rows, int32_t dim, const mux_bf16* a, int64_t lda, const mux_bf16* b, int64_t ldb,
                   mux_bf16* y, int64_t ldy, cudaStream_t stream) {
  mux_status st = ew_check(rows, dim);
  if (st != MUX_OK || rows == 0) return st;
  if (!a || !b || !y) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(a) || !aligned16(b) || !aligned16(y) || !ld_ok(lda, dim) || !ld_ok(ldb, dim) || !ld_ok(ldy, dim))
    return fail(MUX_ERR_INVALID_ARGUMENT, "alignment/stride");
  cudaError_t e = launch_add(rows, dim, a, lda, b, ldb, y, ldy, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_add launch");
  return MUX_OK;
}

// ---------------------------------------------------------------- fused GEMM -> reduce-scatter
mux_status mux_linear_fwd_rs(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task, int32_t num_adapters,
                             const mux_adapter* adapters, int32_t max_rows, int32_t K, int32_t N, int32_t r_cap,
                             const mux_bf16* X_, const mux_bf16* W_, mux_bf16* Hs_, const mux_rs* rs,
                             void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  if (!rs) return fail(MUX_ERR_INVALID_ARGUMENT, "rs is null");
  auto X = reinterpret_cast<const __nv_bfloat16*>(X_);
  return linear_common(false, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap, X, X,
                       reinterpret_cast<const __nv_bfloat16*>(W_), nullptr, nullptr,
                       reinterpret_cast<__nv_bfloat16*>(Hs_), workspace, workspace_bytes, stream, 3, rs);
}

mux_status mux_linear_bwd_dx_rs(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                                int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows, int32_t K,
                                int32_t N, int32_t r_cap, const mux_bf16* dY_, const mux_bf16* X_,
                                const mux_bf16* W_, const mux_bf16* Hs_, const mux_rs* rs, void* workspace,
                                size_t workspace_bytes, cudaStream_t stream) {
  if (!rs) return fail(MUX_ERR_INVALID_ARGUMENT, "rs is null");
  return linear_common(true, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap,
                       reinterpret_cast<const __nv_bfloat16*>(dY_), reinterpret_cast<const __nv_bfloat16*>(X_),
                       reinterpret_cast<const __nv_bfloat16*>(W_), nullptr,
                       reinterpret_cast<const __nv_bfloat16*>(Hs_), nullptr, workspace, workspace_bytes, stream,
                       MUX_BWD_DX, rs);
}

mux_status mux_rs_reduce(const mux_rs* rs, int32_t cols, mux_bf16* out, int64_t ldo, cudaStream_t stream) {
  if (!rs || !out) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (rs->world < 1 || rs->world > MUX_RS_MAX_WORLD || rs->rank < 0 || rs->rank >= rs->world || rs->seq == 0 ||
      rs->rows_per_rank <= 0 || cols < 8 || cols % 8 || !ld_ok(ldo, cols))
    return fail(MUX_ERR_INVALID_ARGUMENT, "rs_reduce: world=%d rank=%d seq=%llu rows=%d cols=%d", rs->world,
                rs->rank, static_cast<unsigned long long>(rs->seq), rs->rows_per_rank, cols);
  for (int d = 0; d < rs->world; ++d)
    if (!rs->flags[d]) return fail(MUX_ERR_INVALID_ARGUMENT, "rs: flags of rank %d null", d);
  if (!rs->recv[rs->rank] || !aligned16(rs->recv[rs->rank]) || !aligned16(out))
    return fail(MUX_ERR_INVALID_ARGUMENT, "rs_reduce: receive buffer / out null or misaligned");
  static thread_local RsReduceParams q;
  q.world = rs->world;
  q.rank = rs->rank;
  q.rows = rs->rows_per_rank;
  q.cols = cols;
  q.seq = rs->seq;
  q.recv = reinterpret_cast<const uint4*>(rs->recv[rs->rank]);
  q.flags = rs->flags[rs->rank];
  for (int s2 = 0; s2 < rs->world; ++s2) q.ack[s2] = rs->flags[s2] + rs->world + rs->rank;
  q.out = reinterpret_cast<uint4*>(out);
  q.ldo8 = ldo / 8;
  q.peer_wait_ns = peer_wait_ns();
  cudaError_t e = launch_rs_reduce(q, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "mux_rs_reduce launch");
  return MUX_OK;
}

size_t mux_rs_flags_elems(int32_t world) { return world > 0 ? static_cast<size_t>(2 * world + 1) : 0; }

// ---------------------------------------------------------------- fused all-gather -> GEMM
mux_status mux_ag_push(const mux_ag* ag, const mux_bf16* rows, int64_t ld, int32_t cols, cudaStream_t stream) {
  if (!ag || !rows) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (ag->world < 1 || ag->world > MUX_RS_MAX_WORLD || ag->rank < 0 || ag->rank >= ag->world || ag->seq == 0 ||
      ag->rows_per_rank <= 0 || cols < 8 || cols % 8 || !ld_ok(ld, cols))
    return fail(MUX_ERR_INVALID_ARGUMENT, "ag_push: world=%d rank=%d rows=%d cols=%d", ag->world, ag->rank,
                ag->rows_per_rank, cols);
  StreamValueFn wait = wait_value64(), write = write_value64();
  if (!wait || !write) return fail(MUX_ERR_UNSUPPORTED, "stream memory operations unavailable");
  const unsigned long long* ack = ag->flags[ag->rank] + ag->world;  // readers' acks, this rank's block
  for (int d = 0; d < ag->world; ++d) {
    if (!ag->recv[d] || !ag->flags[d]) return fail(MUX_ERR_INVALID_ARGUMENT, "ag: rank %d buffers null", d);
    // rank d must have released this rank's rows of the previous call
    if (ag->seq > 1 && wait(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(ack + d),
                            ag->seq - 1, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail(MUX_ERR_CUDA, "cuStreamWaitValue64 failed");
    mux_bf16* dst = ag->recv[d] + static_cast<size_t>(ag->rank) * ag->rows_per_rank * cols;
    cudaError_t e = cudaMemcpy2DAsync(dst, static_cast<size_t>(cols) * 2, rows, static_cast<size_t>(ld) * 2,
                                      static_cast<size_t>(cols) * 2, ag->rows_per_rank, cudaMemcpyDeviceToDevice,
                                      stream);
    if (e != cudaSuccess) return cuda_fail(e, "mux_ag_push copy");
    // ordered after the copy (stream order; the write carries a memory fence)
    if (write(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(ag->flags[d] + ag->rank), ag->seq,
              0) != CUDA_SUCCESS)
      return fail(MUX_ERR_CUDA, "cuStreamWriteValue64 failed");
  }
  return MUX_OK;
}

mux_status mux_ag_release(const mux_ag* ag, cudaStream_t stream) {
  if (!ag) return fail(MUX_ERR_INVALID_ARGUMENT, "null pointer");
  if (ag->world < 1 || ag->world > MUX_RS_MAX_WORLD || ag->rank < 0 || ag->rank >= ag->world || ag->seq == 0)
    return fail(MUX_ERR_INVALID_ARGUMENT, "ag_release: world=%d rank=%d", ag->world, ag->rank);
  StreamValueFn write = write_value64();
  if (!write) return fail(MUX_ERR_UNSUPPORTED, "stream memory operations unavailable");
  for (int s2 = 0; s2 < ag->world; ++s2) {
    if (!ag->flags[s2]) return fail(MUX_ERR_INVALID_ARGUMENT, "ag: rank %d flags null", s2);
    if (write(reinterpret_cast<CUstream>(stream),
              reinterpret_cast<CUdeviceptr>(ag->flags[s2] + ag->world + ag->rank), ag->seq, 0) != CUDA_SUCCESS)
      return fail(MUX_ERR_CUDA, "cuStreamWriteValue64 failed");
  }
  return MUX_OK;
}

mux_status mux_linear_fwd_ag(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task, int32_t num_adapters,
                             const mux_adapter* adapters, int32_t max_rows, int32_t K, int32_t N, int32_t r_cap,
                             const mux_ag* ag, const mux_bf16* W_, mux_bf16* Y_, mux_bf16* Hs_, void* workspace,
                             size_t workspace_bytes, cudaStream_t stream) {
  if (!ag || ag->rank < 0 || ag->rank >= MUX_RS_MAX_WORLD) return fail(MUX_ERR_INVALID_ARGUMENT, "ag is null/bad");
  auto X = reinterpret_cast<const __nv_bfloat16*>(ag->recv[ag->rank]);
  return linear_common(false, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap, X, X,
                       reinterpret_cast<const __nv_bfloat16*>(W_), reinterpret_cast<__nv_bfloat16*>(Y_), nullptr,
                       reinterpret_cast<__nv_bfloat16*>(Hs_), workspace, workspace_bytes, stream, 3, nullptr, ag);
}

mux_status mux_linear_bwd_ag(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task, int32_t num_adapters,
                             const mux_adapter* adapters, int32_t max_rows, int32_t K, int32_t N, int32_t r_cap,
                             const mux_ag* ag, const mux_bf16* X_, const mux_bf16* W_, const mux_bf16* Hs_,
                             mux_bf16* dX_, void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  if (!ag || ag->rank < 0 || ag->rank >= MUX_RS_MAX_WORLD) return fail(MUX_ERR_INVALID_ARGUMENT, "ag is null/bad");
  return linear_common(true, num_segs, seg_off, seg_task, num_adapters, adapters, max_rows, K, N, r_cap,
                       reinterpret_cast<const __nv_bfloat16*>(ag->recv[ag->rank]),
                       reinterpret_cast<const __nv_bfloat16*>(X_), reinterpret_cast<const __nv_bfloat16*>(W_),
                       reinterpret_cast<__nv_bfloat16*>(dX_), reinterpret_cast<const __nv_bfloat16*>(Hs_), nullptr,
                       workspace, workspace_bytes, stream, 3, nullptr, ag);
}

// The generic entry point: every op of the per-op functions above, optionally over column slices
// (mux.h, "Fused projections with one adapter per column slice").
mux_status mux_linear(const mux_linear_args* a) {
  if (!a) return fail(MUX_ERR_INVALID_ARGUMENT, "args is null");
  using bf = __nv_bfloat16;
  auto c = [](const mux_bf16* x) { return reinterpret_cast<const bf*>(x); };
  auto m = [](mux_bf16* x) { return reinterpret_cast<bf*>(x); };
  if (a->ag && (a->ag->rank < 0 || a->ag->rank >= MUX_RS_MAX_WORLD))
    return fail(MUX_ERR_INVALID_ARGUMENT, "ag is bad (rank %d)", a->ag->rank);
  const bf* ag_buf = a->ag ? reinterpret_cast<const bf*>(a->ag->recv[a->ag->rank]) : nullptr;
  switch (a->op) {
    case MUX_OP_FWD: {
      if (a->rs && a->ag) return fail(MUX_ERR_INVALID_ARGUMENT, "fwd: rs and ag together are not supported");
      const bf* X = a->ag ? ag_buf : c(a->X);
      return linear_common(false, a->num_segs, a->seg_off, a->seg_task, a->num_adapters, a->adapters, a->max_rows,
                           a->K, a->N, a->r_cap, X, X, c(a->W), a->rs ? nullptr : m(a->Y), nullptr, m(a->Hs),
                           a->workspace, a->workspace_bytes, a->stream, 3, a->rs, a->ag, false, false, 0, INT32_MAX,
                           a->slices);
    }
    case MUX_OP_FWD_HS:
      if (a->rs || a->ag) return fail(MUX_ERR_INVALID_ARGUMENT, "fwd_hs: no fused collectives");
      if (!a->Hs) return fail(MUX_ERR_INVALID_ARGUMENT, "fwd_hs: Hs (input) is null");
      return linear_common(false, a->num_segs, a->seg_off, a->seg_task, a->num_adapters, a->adapters, a->max_rows,
                           a->K, a->N, a->r_cap, c(a->X), c(a->X), c(a->W), m(a->Y), a->Hs ? c(a->Hs) : nullptr,
                           nullptr, a->workspace, a->workspace_bytes, a->stream, 3, nullptr, nullptr, true, false, 0,
                           INT32_MAX, a->slices);
    case MUX_OP_SHRINK:
      if (a->rs || a->ag) return fail(MUX_ERR_INVALID_ARGUMENT, "shrink: no fused collectives");
      return linear_common(false, a->num_segs, a->seg_off, a->seg_task, a->num_adapters, a->adapters, a->max_rows,
                           a->K, a->N, a->r_cap, c(a->X), c(a->X), nullptr, nullptr, nullptr, m(a->Hs), a->workspace,
                           a->workspace_bytes, a->stream, 3, nullptr, nullptr, false, true, a->row_begin, a->row_end,
                           a->slices);
    case MUX_OP_BWD:
    case MUX_OP_BWD_DX:
    case MUX_OP_BWD_GRADS: {
      const int parts = a->op == MUX_OP_BWD ? 3 : a->op == MUX_OP_BWD_DX ? 1 : 2;
      if (a->rs && a->op != MUX_OP_BWD_DX) return fail(MUX_ERR_INVALID_ARGUMENT, "bwd: rs only with MUX_OP_BWD_DX");
      if (a->rs && a->ag) return fail(MUX_ERR_INVALID_ARGUMENT, "bwd: rs and ag together are not supported");
      const bf* dY = a->ag ? ag_buf : c(a->dY);
      return linear_common(true, a->num_segs, a->seg_off, a->seg_task, a->num_adapters, a->adapters, a->max_rows,
                           a->K, a->N, a->r_cap, dY, c(a->X), c(a->W), a->rs ? nullptr : m(a->dX), c(a->Hs), nullptr,
                           a->workspace, a->workspace_bytes, a->stream, parts, a->rs, a->ag, false, false, 0,
                           INT32_MAX, a->slices, m(a->Gs));
    }
    case MUX_OP_SHRINK_BWD: {
      if (a->rs) return fail(MUX_ERR_INVALID_ARGUMENT, "shrink_bwd: no fused reduce-scatter");
      if (!a->Gs) return fail(MUX_ERR_INVALID_ARGUMENT, "shrink_bwd: Gs (output) is null");
      const bf* dY = a->ag ? ag_buf : c(a->dY);
      return linear_common(true, a->num_segs, a->seg_off, a->seg_task, a->num_adapters, a->adapters, a->max_rows,
                           a->K, a->N, a->r_cap, dY, nullptr, nullptr, nullptr, nullptr, nullptr, a->workspace,
                           a->workspace_bytes, a->stream, 3, nullptr, a->ag, false, true, a->row_begin, a->row_end,
                           a->slices, m(a->Gs));
    }
    default:
      return fail(MUX_ERR_INVALID_ARGUMENT, "unknown op %d", a->op);
  }
}

}  // extern "C"
