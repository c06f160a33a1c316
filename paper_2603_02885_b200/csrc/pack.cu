// pack.cu — chunk-based data alignment (§3.5) as one integer kernel,
// plus the Dispatch gather (token-major rows -> packed rows).
//
// mux_pack_kernel runs as a single 1024-thread CTA (the problem is tiny and
// latency-bound: tens to thousands of sequences; one CTA avoids grid-wide
// syncs and keeps every intermediate in L1/L2):
//   1. chunk size  c = max(chunk_min, 2^{min_s v2(len_s)}) — block min-reduce
//                  of __ffs(len)-1, or the caller's chunk_size;
//   2. per-task order: rank of each sequence in (len desc, index asc) order
//      (counting sort by comparison, all sequences in parallel);
//   3. per-task first-fit decreasing: one warp per task; the first pack
//      with room is found 32 packs at a time with __ballot_sync;
//   4. chunk counts ceil(L_p / c) -> per-task scan -> seg_off, pack rows;
//   5. fill: chunk table with KV-reuse links, seq_row, row_src.
// Integer results are bit-exact with the fp64 oracle's pack (tests/test_gpu_pack.py).
#include <cstdio>

#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

constexpr int kPackThreads = 1024;

// -DMUX_PACK_PROFILE: thread 0 records clock64() at each phase boundary and
// prints the deltas (diagnostic builds only, tools/pack_time.py).
#ifdef MUX_PACK_PROFILE
#define PACK_MARK(i) do { if (threadIdx.x == 0) _pt[i] = clock64(); } while (0)
#else
#define PACK_MARK(i) do { } while (0)
#endif
constexpr int kPackWarps = kPackThreads / 32;

struct PackWs {  // carved from the caller's workspace
  int32_t* order;       // [num_seqs] local index of the r-th sequence of its task in FFD order
  int32_t* pack_of;     // [num_seqs]
  int32_t* pack_off;    // [num_seqs] offset of the sequence inside its pack
  int32_t* residual;    // [num_seqs] per-task packs at [task_seq_off[t] .. ) : residual capacity
  int32_t* pack_len;    // [num_seqs] same indexing: pack length
  int32_t* pack_row0;   // [num_seqs] same indexing: first row of the pack
  int32_t* tok_off;     // [num_seqs + 1] exclusive prefix of lengths
  int32_t* seq_task;    // [num_seqs] task of sequence i (= task of pack slot i)
  int32_t* task_packs;  // [M]
  int32_t* task_chunks; // [M]
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline size_t pack_ws_bytes(int M, int S) {
  const size_t s = align256(sizeof(int32_t) * (size_t)(S + 1));
  return 8 * s + 2 * align256(sizeof(int32_t) * (size_t)(M > 0 ? M : 1));
}

// Shared-memory variant: every per-sequence / per-task array lives in smem
// when it fits (the common case: tens to a few thousand sequences).
constexpr int kPackSmemMaxBytes = 200 * 1024;

__host__ __device__ inline size_t pack_smem_bytes(int M, int S) {
  // workspace arrays + staged copies of seq_len [S], task_seq_off [M+1], capacity [M]
  return 9 * align256(sizeof(int32_t) * (size_t)(S + 1)) + 4 * align256(sizeof(int32_t) * (size_t)(M + 1));
}

__device__ inline PackWs carve_pack_ws(void* ws, int M, int S) {
  uint8_t* b = reinterpret_cast<uint8_t*>(ws);
  const size_t s = align256(sizeof(int32_t) * (size_t)(S + 1));
  const size_t m = align256(sizeof(int32_t) * (size_t)(M > 0 ? M : 1));
  PackWs w;
  w.order = reinterpret_cast<int32_t*>(b); b += s;
  w.pack_of = reinterpret_cast<int32_t*>(b); b += s;
  w.pack_off = reinterpret_cast<int32_t*>(b); b += s;
  w.residual = reinterpret_cast<int32_t*>(b); b += s;
  w.pack_len = reinterpret_cast<int32_t*>(b); b += s;
  w.pack_row0 = reinterpret_cast<int32_t*>(b); b += s;
  w.tok_off = reinterpret_cast<int32_t*>(b); b += s;
  w.seq_task = reinterpret_cast<int32_t*>(b); b += s;
  w.task_packs = reinterpret_cast<int32_t*>(b); b += m;
  w.task_chunks = reinterpret_cast<int32_t*>(b);
  return w;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(kPackThreads, 1)
    mux_pack_kernel(int M, int S, const int32_t* __restrict__ task_seq_off, const int32_t* __restrict__ seq_len,
                    const int32_t* __restrict__ pack_capacity, int chunk_size, int chunk_min, int max_rows,
                    int max_chunks, int32_t* seg_off, int32_t* seq_row, int32_t* chunk_task,
                    int32_t* chunk_pack, int32_t* chunk_valid, int32_t* chunk_dep, int32_t* row_src,
                    mux_pack_info* info, void* workspace, int use_smem) {
  __shared__ int s_red[kPackWarps];
  __shared__ int s_bad, s_ovf, s_c, s_total_chunks, s_maxlen, s_valid;
  extern __shared__ __align__(256) uint8_t pack_smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  PackWs ws = carve_pack_ws(use_smem ? static_cast<void*>(pack_smem) : workspace, M, S);
#ifdef MUX_PACK_PROFILE
  long long _pt[10] = {0};
#endif
  griddep_wait();  // PDL: inputs may come from the previous kernel
  PACK_MARK(0);
  griddep_launch_dependents();
  // Stage the (small) inputs in shared memory when they fit: every later
  // phase re-reads them, and a dependent global round trip per phase was the
  // kernel's critical path.
  const int32_t* sl = seq_len;
  const int32_t* tso = task_seq_off;
  const int32_t* capp = pack_capacity;
  if (use_smem) {
    uint8_t* b = pack_smem + 8 * align256(sizeof(int32_t) * (size_t)(S + 1)) +
                 2 * align256(sizeof(int32_t) * (size_t)(M > 0 ? M : 1));
    int32_t* s_sl = reinterpret_cast<int32_t*>(b);
    b += align256(sizeof(int32_t) * (size_t)(S + 1));
    int32_t* s_tso = reinterpret_cast<int32_t*>(b);
    b += align256(sizeof(int32_t) * (size_t)(M + 1));
    int32_t* s_cap = reinterpret_cast<int32_t*>(b);
    for (int i = tid; i < S; i += kPackThreads) s_sl[i] = seq_len[i];
    for (int i = tid; i <= M; i += kPackThreads) s_tso[i] = task_seq_off[i];
    if (pack_capacity != nullptr)
      for (int i = tid; i < M; i += kPackThreads) s_cap[i] = pack_capacity[i];
    __syncthreads();
    sl = s_sl;
    tso = s_tso;
    capp = pack_capacity != nullptr ? s_cap : nullptr;
  }

  PACK_MARK(1);
  // ---- 1. chunk size, validity, max length, valid rows -------------------
  int v2min = 30, bad = 0, mx = 0, sum = 0;
  for (int i = tid; i < S; i += kPackThreads) {
    const int L = sl[i];
    if (L < 1) bad = 1;
    else {
      v2min = min(v2min, __ffs(L) - 1);
      mx = max(mx, L);
      sum += L;
    }
  }
  if (tid == 0) { s_bad = 0; s_maxlen = 0; s_valid = 0; }
  __syncthreads();
  v2min = warp_min(v2min);
  if (lane == 0) s_red[warp] = v2min;
  mx = warp_max(mx);
  sum = warp_sum(sum);
  if (lane == 0) { atomicMax(&s_maxlen, mx); atomicAdd(&s_valid, sum); }
  if (bad) s_bad = 4;
  __syncthreads();
  if (warp == 0) {
    int v = s_red[lane];
    v = warp_min(v);
    if (lane == 0) {
      int c = chunk_size;
      if (c == 0) c = (S == 0) ? chunk_min : max(chunk_min, 1 << v);
      s_c = c;
    }
  }
  __syncthreads();
  const int c = s_c;
  if (s_bad) {
    if (tid == 0) {
      mux_pack_info r{};
      r.chunk_size = c;
      r.overflow = s_bad;
      *info = r;
    }
    return;
  }

  PACK_MARK(2);
  // ---- 2. FFD visit order per task: rank by (len desc, index asc) ---------
  for (int i = tid; i < S; i += kPackThreads) {
    // task of sequence i: binary search in task_seq_off
    int lo = 0, hi = M;  // find t with off[t] <= i < off[t+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (tso[mid] <= i) lo = mid; else hi = mid;
    }
    const int t0 = tso[lo], t1 = tso[lo + 1];
    ws.seq_task[i] = lo;
    const int L = sl[i];
    int rank = 0;
    for (int j = t0; j < t1; ++j) {
      const int Lj = sl[j];
      rank += (Lj > L) || (Lj == L && j < i);
    }
    ws.order[t0 + rank] = i - t0;
  }
  __syncthreads();

  PACK_MARK(3);
  // ---- 3. first-fit decreasing, one warp per task -------------------------
  for (int t = warp; t < M; t += kPackWarps) {
    const int t0 = tso[t], n = tso[t + 1] - t0;
    int mxl = 0;
    for (int i = lane; i < n; i += 32) mxl = max(mxl, sl[t0 + i]);
    mxl = warp_max(mxl);
    int cap;
    if (capp != nullptr) cap = capp[t];
    else cap = ((max(mxl, c) + c - 1) / c) * c;
    if (n > 0 && cap < mxl) {
      if (lane == 0) atomicOr(&s_bad, 4);
      continue;
    }
    int* resid = ws.residual + t0;
    int npacks = 0;
    for (int r = 0; r < n; ++r) {
      const int li = ws.order[t0 + r];
      const int L = sl[t0 + li];
      int found = -1;
      for (int base = 0; base < npacks && found < 0; base += 32) {
        const int p = base + lane;
        const bool fits = p < npacks && resid[p] >= L;
        const unsigned bal = __ballot_sync(0xffffffffu, fits);
        if (bal) found = base + __ffs(bal) - 1;
      }
      if (found < 0) {
        found = npacks++;
        if (lane == 0) resid[found] = cap;
      }
      __syncwarp();
      if (lane == 0) {
        ws.pack_of[t0 + li] = found;
        ws.pack_off[t0 + li] = cap - resid[found];
        resid[found] -= L;
      }
      __syncwarp();
    }
    // pack lengths and chunk counts
    int nch = 0;
    for (int p = lane; p < npacks; p += 32) {
      const int len = cap - resid[p];
      ws.pack_len[t0 + p] = len;
      nch += (len + c - 1) / c;
    }
    nch = warp_sum(nch);
    if (lane == 0) {
      ws.task_packs[t] = npacks;
      ws.task_chunks[t] = nch;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) {
      mux_pack_info r{};
      r.chunk_size = c;
      r.overflow = s_bad;
      *info = r;
    }
    return;
  }

  PACK_MARK(4);
  // ---- 4. scan over tasks -> seg_off; overflow check ----------------------
  if (warp == 0) {  // exclusive prefix of chunk counts, 32 tasks at a time
    int acc = 0, packs = 0;
    for (int base = 0; base < M; base += 32) {
      const int t = base + lane;
      const int v = t < M ? ws.task_chunks[t] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (t < M) ws.task_chunks[t] = acc + x - v;
      acc += __shfl_sync(0xffffffffu, x, 31);
      packs += warp_sum(t < M ? ws.task_packs[t] : 0);
    }
    if (lane == 0) {
      s_total_chunks = acc;
      int ovf = 0;
      if (acc * c > max_rows) ovf |= 1;
      if (acc > max_chunks) ovf |= 2;
      mux_pack_info r;
      r.chunk_size = c;
      r.num_chunks = acc;
      r.num_packs = packs;
      r.total_rows = acc * c;
      r.valid_rows = s_valid;
      r.zero_pad_rows = S * s_maxlen;
      r.overflow = ovf;
      *info = r;
      s_ovf = ovf;  // separate flag: other threads may still be reading s_bad above
    }
  }
  __syncthreads();
  if (s_ovf) return;
  const int total_chunks = s_total_chunks;
  for (int t = tid; t <= M; t += kPackThreads) seg_off[t] = (t < M ? ws.task_chunks[t] : total_chunks) * c;

  // per-task pack rows (serial over a task's packs; one warp per task)
  for (int t = warp; t < M; t += kPackWarps) {
    if (lane == 0) {
      const int t0 = tso[t];
      int ch = ws.task_chunks[t];
      for (int p = 0; p < ws.task_packs[t]; ++p) {
        ws.pack_row0[t0 + p] = ch * c;
        ch += (ws.pack_len[t0 + p] + c - 1) / c;
      }
    }
  }
  // token offsets: exclusive prefix over all sequences (warp 0, 32 at a time)
  if (warp == 0) {
    int run = 0;
    for (int base = 0; base < S; base += 32) {
      const int i = base + lane;
      int v = i < S ? sl[i] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < S) ws.tok_off[i] = run + x - v;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  // rows past the last chunk are unused
  for (int r = total_chunks * c + tid; r < max_rows; r += kPackThreads) row_src[r] = -1;
  __syncthreads();

  PACK_MARK(5);
  // ---- 5. fill ------------------------------------------------------------
  // Flat over all tasks at once (a serial loop over tasks was the kernel's
  // critical path at 16-32 tasks): one warp per pack slot, then one warp per
  // sequence; the lanes write a pack's chunks / tail rows and a sequence's
  // rows in parallel.  Pack slot j of task t is ws.*[tso[t] + p], p < task_packs[t].
  for (int j = warp; j < S; j += kPackWarps) {
    const int t = ws.seq_task[j];
    const int p = j - tso[t];
    if (p >= ws.task_packs[t]) continue;
    const int len = ws.pack_len[j];
    const int n_p = (len + c - 1) / c;
    const int id0 = ws.pack_row0[j] / c;
    for (int q = lane; q < n_p; q += 32) {
      chunk_task[id0 + q] = t;
      chunk_pack[id0 + q] = p;
      chunk_valid[id0 + q] = min(c, len - q * c);
      chunk_dep[id0 + q] = q > 0 ? id0 + q - 1 : -1;
    }
    // the pack's tail padding (its sequences fill [row0, row0 + len))
    for (int r = id0 * c + len + lane; r < (id0 + n_p) * c; r += 32) row_src[r] = -1;
  }
  // seq_row and row_src: one warp per sequence
  for (int s = warp; s < S; s += kPackWarps) {
    const int row = ws.pack_row0[tso[ws.seq_task[s]] + ws.pack_of[s]] + ws.pack_off[s];
    if (lane == 0) seq_row[s] = row;
    const int L = sl[s];
    const int tok = ws.tok_off[s];
    // head up to a 16-byte boundary, then 4 rows per lane per int4 store, then the tail
    const int head = min(L, static_cast<int>(((16u - (reinterpret_cast<uintptr_t>(row_src + row) & 15u)) & 15u) >> 2));
    if (lane < head) row_src[row + lane] = tok + lane;
    const int nvec = (L - head) >> 2;
    int4* body = reinterpret_cast<int4*>(row_src + row + head);
    for (int q = lane; q < nvec; q += 32) {
      const int v = tok + head + 4 * q;
      body[q] = make_int4(v, v + 1, v + 2, v + 3);
    }
    const int done = head + 4 * nvec;
    if (done + lane < L) row_src[row + done + lane] = tok + done + lane;
  }
#ifdef MUX_PACK_PROFILE
  __syncthreads();
  PACK_MARK(6);
  if (threadIdx.x == 0)
    printf("pack_profile M=%d S=%d cycles: stage %lld chunk %lld order %lld ffd %lld scan+rows %lld fill %lld\n", M, S,
           _pt[1] - _pt[0], _pt[2] - _pt[1], _pt[3] - _pt[2], _pt[4] - _pt[3], _pt[5] - _pt[4], _pt[6] - _pt[5]);
#endif
}

// Dispatch gather: 16-byte vectors, one warp-row at a time.
__global__ void mux_pack_apply_kernel(int max_rows, int cols, int num_tokens, const int32_t* __restrict__ row_src,
                                      const uint4* __restrict__ src, uint4* __restrict__ dst) {
  griddep_wait();
  griddep_launch_dependents();
  const int vec_per_row = cols / 8;
  const long long total = static_cast<long long>(max_rows) * vec_per_row;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx / vec_per_row);
    const int v = static_cast<int>(idx - static_cast<long long>(r) * vec_per_row);
    const int s = row_src[r];
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (s >= 0 && s < num_tokens) val = src[static_cast<long long>(s) * vec_per_row + v];
    dst[idx] = val;
  }
}

size_t pack_workspace_bytes(int M, int S) { return pack_ws_bytes(M, S); }

cudaError_t launch_pack(int M, int S, const int32_t* task_seq_off, const int32_t* seq_len,
                        const int32_t* pack_capacity, int chunk_size, int chunk_min, int max_rows, int max_chunks,
                        int32_t* seg_off, int32_t* seq_row, int32_t* chunk_task, int32_t* chunk_pack,
                        int32_t* chunk_valid, int32_t* chunk_dep, int32_t* row_src, mux_pack_info* info,
                        void* workspace, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t ce = once_per_device(configured, [] {
    return cudaFuncSetAttribute(mux_pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPackSmemMaxBytes);
  });
  if (ce != cudaSuccess) return ce;
  const size_t smem = pack_smem_bytes(M, S);
  const int use_smem = smem <= static_cast<size_t>(kPackSmemMaxBytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kPackThreads);
  cfg.dynamicSmemBytes = use_smem ? smem : 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mux_pack_kernel, M, S, task_seq_off, seq_len, pack_capacity, chunk_size, chunk_min,
                            max_rows, max_chunks, seg_off, seq_row, chunk_task, chunk_pack, chunk_valid, chunk_dep,
                            row_src, info, workspace, use_smem);
}

cudaError_t launch_pack_apply(int max_rows, int cols, int num_tokens, const int32_t* row_src,
                              const __nv_bfloat16* src, __nv_bfloat16* dst, int num_sms, cudaStream_t stream) {
  const long long total = static_cast<long long>(max_rows) * (cols / 8);
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  const long long cap = static_cast<long long>(num_sms) * 8;
  if (blocks > cap) blocks = cap;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mux_pack_apply_kernel, max_rows, cols, num_tokens, row_src,
                            reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst));
}

}  // namespace mux

namespace mux {
// Debug builds (-DMUX_DEBUG_CHECKS): the device-side preconditions of the
// linear calls that the host cannot check without a synchronisation
// (include/mux.h): seg_off non-decreasing, every entry a multiple of 64,
// seg_off[S] <= max_rows.  A violation prints the offending entry and traps.
__global__ void mux_check_segments_kernel(int num_segs, const int32_t* seg_off, int max_rows) {
  griddep_wait();
  griddep_launch_dependents();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int s = 0; s <= num_segs; ++s) {
    const int v = seg_off[s];
    const bool bad = (v % kRowQuarter) != 0 || v < 0 || v > max_rows || (s > 0 && v < seg_off[s - 1]);
    if (bad) {
      printf("mux: bad seg_off[%d] = %d (max_rows %d): must be non-decreasing multiples of 64 <= max_rows\n", s,
             v, max_rows);
      __trap();
    }
  }
}

cudaError_t launch_check_segments(int num_segs, const int32_t* seg_off, int max_rows, cudaStream_t s) {
  return launch_pdl(mux_check_segments_kernel, dim3(1), dim3(32), 0, s, num_segs, seg_off, max_rows);
}
}  // namespace mux
