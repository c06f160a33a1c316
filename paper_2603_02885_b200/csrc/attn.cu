// attn.cu — backward of the causal attention inside packed sequences (the
// forward is attn_tc.cu, on tcgen05):
// the chunk dependency of the paper's alignment ("KV cache reuse in causal
// attention", Fig. alignment): the queries of a chunk attend to the
// keys of the earlier chunks of the same pack, masked to their own sequence
// (packing without that mask "wastes attention computation across sequences",
// P:810-811).  With row_start[r] = first row of r's sequence (-1 = pad):
//     o_r = sum_{j = row_start[r] .. r} softmax_j(scale <q_r, k_j>) v_j.
//
// Flash-attention style: S and P never reach HBM.  Head dim 128 (every
// LLaMA size), grouped KV heads (H % Hkv == 0, LLaMA-70B's k/v).  Tiles of 64
// rows; each warp owns 16 rows and runs warp-level bf16 tensor-core MMAs
// (mma.sync m16n8k16, fp32 accumulate) on ldmatrix fragments of 128 B-
// swizzled shared-memory tiles fed by cp.async double buffering.  At the
// paper's sequence lengths (<= 512) attention is < 1% of a decoder block's
// FLOPs, so this warp-level design, not tcgen05, is used here.
//   bwd : D = rowsum(dO * O); dK, dV per key tile (loops over the query tiles
//         that see it and over the q heads of its KV group); dQ per query tile
//         — two kernels, no atomics: deterministic.
#include <algorithm>
#include <climits>
#include <cmath>

#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

constexpr int kHd = 128;                  // head dim
constexpr int kRowB = kHd * 2;            // 256 B per smem row
constexpr int kAttnThreads = 128;         // 4 warps x 16 rows
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>(row * kRowB + ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Fragment loads from a swizzled [rows][128] bf16 tile at smem address `t`:
// A (16 x 16 at row0, k0; rows = M, cols = K)
__device__ __forceinline__ void ld_a(uint32_t t, int row0, int k0, int lane, uint32_t (&a)[4]) {
  const int j = lane >> 3;
  ldsm_x4(t + swz(row0 + (lane & 7) + (j & 1) * 8, (k0 >> 3) + (j >> 1)), a[0], a[1], a[2], a[3]);
}
// B for two n8 tiles (n0, n0+8) at k0 from a tile stored [n][k] (non-transposed)
__device__ __forceinline__ void ld_b(uint32_t t, int n0, int k0, int lane, uint32_t (&b)[4]) {
  const int j = lane >> 3;
  ldsm_x4(t + swz(n0 + (lane & 7) + (j >> 1) * 8, (k0 >> 3) + (j & 1)), b[0], b[1], b[2], b[3]);
}
// B for two n8 tiles (n0, n0+8) at k0 from a tile stored [k][n] (transposed load)
__device__ __forceinline__ void ld_bt(uint32_t t, int k0, int n0, int lane, uint32_t (&b)[4]) {
  const int j = lane >> 3;
  ldsm_x4_t(t + swz(k0 + (lane & 7) + (j & 1) * 8, (n0 >> 3) + (j >> 1)), b[0], b[1], b[2], b[3]);
}
// C fragments of two adjacent n8 tiles -> the A fragment of one k16 step
__device__ __forceinline__ void c_to_a(const float (&c0)[4], const float (&c1)[4], uint32_t (&a)[4]) {
  a[0] = pack_bf16x2(c0[0], c0[1]);
  a[1] = pack_bf16x2(c0[2], c0[3]);
  a[2] = pack_bf16x2(c1[0], c1[1]);
  a[3] = pack_bf16x2(c1[2], c1[3]);
}

// rows [r0, r0 + kRows) of a [R, ld] bf16 matrix (columns col0 .. col0+127) -> swizzled smem; rows >= R are 0
template <int kRows>
__device__ __forceinline__ void load_tile(uint32_t t, const __nv_bfloat16* base, long long ld, int r0, int R) {
  for (int i = threadIdx.x; i < kRows * 16; i += blockDim.x) {
    const int row = i >> 4, ch = i & 15;
    const int r = r0 + row;
    const bool ok = r >= 0 && r < R;
    cp_async16(t + swz(row, ch), base + static_cast<long long>(ok ? r : 0) * ld + ch * 8, ok);
  }
}

__device__ __forceinline__ float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// key range [lo, hi] seen by the 64 query rows q0.. (lo = min row_start over
// valid rows, hi = last valid row); hi = -1 if the tile holds only pads.
__device__ __forceinline__ void tile_key_range(const int32_t* row_start, int q0, int R, int* s_lo, int* s_hi) {
  if (threadIdx.x < 32) {
    int lo = INT_MAX, hi = -1;
    for (int i = threadIdx.x; i < 64; i += 32) {
      const int r = q0 + i;
      if (r < R) {
        const int rs = row_start[r];
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
    if (threadIdx.x == 0) {
      *s_lo = lo;
      *s_hi = hi;
    }
  }
  __syncthreads();
}

// =========================================================================== backward
// D[r, h] = sum_d dO[r, h, d] O[r, h, d]  (one warp per (row, head))
__global__ void __launch_bounds__(256) mux_attn_bwd_pre_kernel(int R, int H, const __nv_bfloat16* dO,
                                                              long long lddo, const __nv_bfloat16* O,
                                                              long long ldo, float* D) {
  griddep_wait();
  griddep_launch_dependents();
  const long long wid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= static_cast<long long>(R) * H) return;
  const long long r = wid / H;
  const int h = static_cast<int>(wid - r * H);
  const uint2 a = *reinterpret_cast<const uint2*>(dO + r * lddo + h * kHd + lane * 4);
  const uint2 b = *reinterpret_cast<const uint2*>(O + r * ldo + h * kHd + lane * 4);
  float acc = __uint_as_float(a.x << 16) * __uint_as_float(b.x << 16) +
              __uint_as_float(a.x & 0xFFFF0000u) * __uint_as_float(b.x & 0xFFFF0000u) +
              __uint_as_float(a.y << 16) * __uint_as_float(b.y << 16) +
              __uint_as_float(a.y & 0xFFFF0000u) * __uint_as_float(b.y & 0xFFFF0000u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) D[wid] = acc;
}

// dK, dV of a 64-key tile of KV head hk: grid (ceil(R/64), Hkv).
// smem: K 16 KB | V 16 KB | 2 x (Q 8 KB, dO 8 KB) | 2 x 32 x {lse2, D, row_start}
constexpr int kBQ = 32;  // query rows per inner step
__global__ void __launch_bounds__(kAttnThreads) mux_attn_bwd_dkdv_kernel(
    int R, int H, int Hkv, const __nv_bfloat16* q, long long ldq, const __nv_bfloat16* k, long long ldk,
    const __nv_bfloat16* v, long long ldv, const __nv_bfloat16* dO, long long lddo, const float* lse,
    const float* Dv, const int32_t* row_start, float scale_log2, float scale, __nv_bfloat16* dk, long long lddk,
    __nv_bfloat16* dv, long long lddv) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ int s_first, s_last, s_qend;
  __shared__ float s_lse[2][kBQ], s_D[2][kBQ];
  __shared__ int s_rs[2][kBQ];
  griddep_wait();
  griddep_launch_dependents();
  const int k0 = blockIdx.x * 64;
  const int hk = blockIdx.y;
  const int G = H / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t sK = smem_u32(smem), sV = sK + 64 * kRowB, sQ0 = sV + 64 * kRowB;
  constexpr uint32_t kQBuf = 2 * kBQ * kRowB;  // Q + dO per buffer
  // valid keys of the tile and the end of the last one's sequence
  if (threadIdx.x < 32) {
    int first = INT_MAX, last = -1;
    for (int i = lane; i < 64; i += 32) {
      const int r = k0 + i;
      if (r < R && row_start[r] >= 0) {
        first = min(first, r);
        last = max(last, r);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
      last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    }
    int qend = last;
    if (last >= 0) {
      const int s = row_start[last];
      for (int base = last + 1; base < R; base += 32) {
        const int r = base + lane;
        const bool same = r < R && row_start[r] == s;
        const unsigned m = __ballot_sync(0xffffffffu, same);
        if (m != 0xffffffffu) {
          qend = base + __ffs(~m) - 2;
          break;
        }
        qend = base + 31;
      }
      qend = min(qend, R - 1);
    }
    if (lane == 0) {
      s_first = first;
      s_last = last;
      s_qend = qend;
    }
  }
  __syncthreads();
  const int first = s_first, qend = s_qend;
  const int kr0 = k0 + warp * 16 + g, kr1 = kr0 + 8;  // this thread's key rows
  float dka[16][4], dva[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dka[i][e] = dva[i][e] = 0.f;
  if (s_last >= 0) {
    load_tile<64>(sK, k + hk * kHd, ldk, k0, R);
    load_tile<64>(sV, v + hk * kHd, ldv, k0, R);
    cp_async_commit();
    const int nq = (qend - first) / kBQ + 1;  // query tiles per head
    const int steps = nq * G;
    auto issue = [&](int step) {
      const int hh = step / nq, qi = step - hh * nq;
      const int h = hk * G + hh;
      const int qt = first + qi * kBQ;
      const int b = step & 1;
      const uint32_t bq = sQ0 + b * kQBuf;
      load_tile<kBQ>(bq, q + h * kHd, ldq, qt, R);
      load_tile<kBQ>(bq + kBQ * kRowB, dO + h * kHd, lddo, qt, R);
      if (threadIdx.x < kBQ) {
        const int r = qt + threadIdx.x;
        const bool ok = r < R;
        s_lse[b][threadIdx.x] = ok ? lse[static_cast<long long>(r) * H + h] * kLog2e : INFINITY;
        s_D[b][threadIdx.x] = ok ? Dv[static_cast<long long>(r) * H + h] : 0.f;
        s_rs[b][threadIdx.x] = ok ? row_start[r] : -1;
      }
      cp_async_commit();
    };
    issue(0);
    for (int step = 0; step < steps; ++step) {
      const int qi = step % nq;
      const int qt = first + qi * kBQ;
      const int b = step & 1;
      if (step + 1 < steps) {
        __syncthreads();  // buffer b^1 free (consumed two steps ago) and its scalars
        issue(step + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const uint32_t bq = sQ0 + b * kQBuf, bdo = bq + kBQ * kRowB;
      // S^T = K Q^T (16 keys x 32 queries per warp), dP^T = V dO^T
      float st[4][4], dpt[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t ak[4], av[4];
        ld_a(sK, warp * 16, ks * 16, lane, ak);
        ld_a(sV, warp * 16, ks * 16, lane, av);
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          uint32_t bq4[4], bd4[4];
          ld_b(bq, np * 16, ks * 16, lane, bq4);
          ld_b(bdo, np * 16, ks * 16, lane, bd4);
          mma16816(st[2 * np], ak, bq4[0], bq4[1]);
          mma16816(st[2 * np + 1], ak, bq4[2], bq4[3]);
          mma16816(dpt[2 * np], av, bd4[0], bd4[1]);
          mma16816(dpt[2 * np + 1], av, bd4[2], bd4[3]);
        }
      }
      // P^T and dS^T (columns = queries)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = nt * 8 + 2 * t4 + e;
          const int qr = qt + c;
          const int rs = s_rs[b][c];
          const float l2 = s_lse[b][c], dd = s_D[b][c];
          const bool v0 = rs >= 0 && rs <= kr0 && kr0 <= qr;
          const bool v1 = rs >= 0 && rs <= kr1 && kr1 <= qr;
          const float p0 = v0 ? exp2f(st[nt][e] * scale_log2 - l2) : 0.f;
          const float p1 = v1 ? exp2f(st[nt][2 + e] * scale_log2 - l2) : 0.f;
          st[nt][e] = p0;
          st[nt][2 + e] = p1;
          dpt[nt][e] = p0 * (dpt[nt][e] - dd);
          dpt[nt][2 + e] = p1 * (dpt[nt][2 + e] - dd);
        }
      }
      // dV += P^T dO,  dK += dS^T Q   (k = 32 queries, n = 128 dims)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        uint32_t ap[4], as[4];
        c_to_a(st[2 * kk], st[2 * kk + 1], ap);
        c_to_a(dpt[2 * kk], dpt[2 * kk + 1], as);
#pragma unroll
        for (int dn = 0; dn < 8; ++dn) {
          uint32_t bd[4], bqq[4];
          ld_bt(bdo, kk * 16, dn * 16, lane, bd);
          ld_bt(bq, kk * 16, dn * 16, lane, bqq);
          mma16816(dva[2 * dn], ap, bd[0], bd[1]);
          mma16816(dva[2 * dn + 1], ap, bd[2], bd[3]);
          mma16816(dka[2 * dn], as, bqq[0], bqq[1]);
          mma16816(dka[2 * dn + 1], as, bqq[2], bqq[3]);
        }
      }
    }
  }
#pragma unroll
  for (int dn = 0; dn < 16; ++dn) {
    const int col = hk * kHd + dn * 8 + 2 * t4;
    if (kr0 < R) {
      *reinterpret_cast<uint32_t*>(dk + static_cast<long long>(kr0) * lddk + col) =
          pack_bf16x2(dka[dn][0] * scale, dka[dn][1] * scale);
      *reinterpret_cast<uint32_t*>(dv + static_cast<long long>(kr0) * lddv + col) =
          pack_bf16x2(dva[dn][0], dva[dn][1]);
    }
    if (kr1 < R) {
      *reinterpret_cast<uint32_t*>(dk + static_cast<long long>(kr1) * lddk + col) =
          pack_bf16x2(dka[dn][2] * scale, dka[dn][3] * scale);
      *reinterpret_cast<uint32_t*>(dv + static_cast<long long>(kr1) * lddv + col) =
          pack_bf16x2(dva[dn][2], dva[dn][3]);
    }
  }
}

// dQ of a 64-query tile of head h: grid (ceil(R/64), H).
// smem: Q 16 KB | dO 16 KB | 2 x (K 16 KB, V 16 KB)
__global__ void __launch_bounds__(kAttnThreads) mux_attn_bwd_dq_kernel(
    int R, int H, int Hkv, const __nv_bfloat16* q, long long ldq, const __nv_bfloat16* k, long long ldk,
    const __nv_bfloat16* v, long long ldv, const __nv_bfloat16* dO, long long lddo, const float* lse,
    const float* Dv, const int32_t* row_start, float scale_log2, float scale, __nv_bfloat16* dq, long long lddq) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ int s_lo, s_hi;
  griddep_wait();
  griddep_launch_dependents();
  const int q0 = blockIdx.x * 64;
  const int h = blockIdx.y;
  const int hk = h / (H / Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t sQ = smem_u32(smem), sdO = sQ + 64 * kRowB, sKV = sdO + 64 * kRowB;
  tile_key_range(row_start, q0, R, &s_lo, &s_hi);
  const int lo = s_lo, hi = s_hi;
  const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;
  const int lo0 = r0 < R ? row_start[r0] : -1, lo1 = r1 < R ? row_start[r1] : -1;
  const float l20 = lo0 >= 0 ? lse[static_cast<long long>(r0) * H + h] * kLog2e : 0.f;
  const float l21 = lo1 >= 0 ? lse[static_cast<long long>(r1) * H + h] * kLog2e : 0.f;
  const float D0 = lo0 >= 0 ? Dv[static_cast<long long>(r0) * H + h] : 0.f;
  const float D1 = lo1 >= 0 ? Dv[static_cast<long long>(r1) * H + h] : 0.f;
  float dqa[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) dqa[i][0] = dqa[i][1] = dqa[i][2] = dqa[i][3] = 0.f;
  if (hi >= 0) {
    load_tile<64>(sQ, q + h * kHd, ldq, q0, R);
    load_tile<64>(sdO, dO + h * kHd, lddo, q0, R);
    load_tile<64>(sKV, k + hk * kHd, ldk, lo, R);
    load_tile<64>(sKV + 64 * kRowB, v + hk * kHd, ldv, lo, R);
    cp_async_commit();
    const int ntiles = (hi - lo) / 64 + 1;
    for (int it = 0; it < ntiles; ++it) {
      const int kt = lo + it * 64;
      const uint32_t sK = sKV + (it & 1) * (128 * kRowB), sV = sK + 64 * kRowB;
      if (it + 1 < ntiles) {
        const uint32_t nK = sKV + ((it + 1) & 1) * (128 * kRowB);
        load_tile<64>(nK, k + hk * kHd, ldk, kt + 64, R);
        load_tile<64>(nK + 64 * kRowB, v + hk * kHd, ldv, kt + 64, R);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      float s[8][4], dp[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t aq[4], ad[4];
        ld_a(sQ, warp * 16, ks * 16, lane, aq);
        ld_a(sdO, warp * 16, ks * 16, lane, ad);
#pragma unroll
        for (int np = 0; np < 4; ++np) {
          uint32_t bk[4], bv[4];
          ld_b(sK, np * 16, ks * 16, lane, bk);
          ld_b(sV, np * 16, ks * 16, lane, bv);
          mma16816(s[2 * np], aq, bk[0], bk[1]);
          mma16816(s[2 * np + 1], aq, bk[2], bk[3]);
          mma16816(dp[2 * np], ad, bv[0], bv[1]);
          mma16816(dp[2 * np + 1], ad, bv[2], bv[3]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = kt + nt * 8 + 2 * t4 + e;
          const bool v0 = lo0 >= 0 && j >= lo0 && j <= r0;
          const bool v1 = lo1 >= 0 && j >= lo1 && j <= r1;
          const float p0 = v0 ? exp2f(s[nt][e] * scale_log2 - l20) : 0.f;
          const float p1 = v1 ? exp2f(s[nt][2 + e] * scale_log2 - l21) : 0.f;
          s[nt][e] = p0 * (dp[nt][e] - D0);
          s[nt][2 + e] = p1 * (dp[nt][2 + e] - D1);
        }
      }
      // dQ += dS K  (k = 64 keys, n = 128 dims)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t a[4];
        c_to_a(s[2 * kk], s[2 * kk + 1], a);
#pragma unroll
        for (int dn = 0; dn < 8; ++dn) {
          uint32_t b[4];
          ld_bt(sK, kk * 16, dn * 16, lane, b);
          mma16816(dqa[2 * dn], a, b[0], b[1]);
          mma16816(dqa[2 * dn + 1], a, b[2], b[3]);
        }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int dn = 0; dn < 16; ++dn) {
    const int col = h * kHd + dn * 8 + 2 * t4;
    if (r0 < R)
      *reinterpret_cast<uint32_t*>(dq + static_cast<long long>(r0) * lddq + col) =
          pack_bf16x2(dqa[dn][0] * scale, dqa[dn][1] * scale);
    if (r1 < R)
      *reinterpret_cast<uint32_t*>(dq + static_cast<long long>(r1) * lddq + col) =
          pack_bf16x2(dqa[dn][2] * scale, dqa[dn][3] * scale);
  }
}

// ------------------------------------------------------------------ launchers
constexpr size_t kDkdvSmem = 2 * 64 * kRowB + 2 * 2 * kBQ * kRowB;  // 64 KB
constexpr size_t kDqSmem = 6 * 64 * kRowB;                    // 96 KB

cudaError_t launch_attn_bwd(int R, int H, int Hkv, const void* dO, long long lddo, const void* q, long long ldq,
                            const void* k, long long ldk, const void* v, long long ldv, const void* o,
                            long long ldo, const float* lse, const int32_t* row_start, float scale, void* dq,
                            long long lddq, void* dk, long long lddk, void* dv, long long lddv, float* Dws,
                            cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(mux_attn_bwd_dkdv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kDkdvSmem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mux_attn_bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kDqSmem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (R == 0) return cudaSuccess;
  const auto b = [](const void* p) { return static_cast<const __nv_bfloat16*>(p); };
  const long long warps = static_cast<long long>(R) * H;
  cudaError_t e = launch_pdl(mux_attn_bwd_pre_kernel, dim3(static_cast<unsigned>((warps + 7) / 8)), dim3(256), 0,
                             s, R, H, b(dO), lddo, b(o), ldo, Dws);
  if (e != cudaSuccess) return e;
  e = launch_pdl(mux_attn_bwd_dkdv_kernel, dim3((R + 63) / 64, Hkv), dim3(kAttnThreads), kDkdvSmem, s, R, H, Hkv,
                 b(q), ldq, b(k), ldk, b(v), ldv, b(dO), lddo, lse, static_cast<const float*>(Dws), row_start,
                 scale * kLog2e, scale, static_cast<__nv_bfloat16*>(dk), lddk, static_cast<__nv_bfloat16*>(dv),
                 lddv);
  if (e != cudaSuccess) return e;
  return launch_pdl(mux_attn_bwd_dq_kernel, dim3((R + 63) / 64, H), dim3(kAttnThreads), kDqSmem, s, R, H, Hkv,
                    b(q), ldq, b(k), ldk, b(v), ldv, b(dO), lddo, lse, static_cast<const float*>(Dws), row_start,
                    scale * kLog2e, scale, static_cast<__nv_bfloat16*>(dq), lddq);
}

}  // namespace mux
