// block.cu — the HBM-bound decoder-block ops around the multiplexed linears
// (SURVEY §8(f) NEXT-3): packed-row sequence map, RMSNorm, SwiGLU, RoPE.
// LLaMA definitions (the backbones of the paper's workloads); the
// backbone is frozen, so RMSNorm's weight gets no gradient.  Every
// kernel moves 16-byte vectors (8 bf16) and accumulates in fp32.
#include <algorithm>
#include <cmath>

#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

// ------------------------------------------------------------------ row map
// row_start[r] = first packed row of r's sequence, -1 for pad rows (the
// chunk layout of P:837: a sequence occupies consecutive rows of its pack).
__global__ void __launch_bounds__(256) mux_row_fill_kernel(int32_t* row_start, int n) {
  griddep_wait();
  griddep_launch_dependents();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) row_start[i] = -1;
}

__global__ void __launch_bounds__(256) mux_row_scatter_kernel(int num_seqs, const int32_t* seq_len,
                                                             const int32_t* seq_row, int32_t* row_start,
                                                             int max_rows) {
  griddep_wait();
  griddep_launch_dependents();
  for (int s = blockIdx.x; s < num_seqs; s += gridDim.x) {
    const int a = seq_row[s];
    const int L = seq_len[s];
    for (int i = threadIdx.x; i < L; i += blockDim.x)
      if (a + i < max_rows) row_start[a + i] = a;
  }
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float (&f)[8]) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                    pack_bf16x2(f[6], f[7]));
}

template <int kThreads>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

// ------------------------------------------------------------------ RMSNorm
// One CTA per row, fp32 sums.  The pre-norm residual stream is fused in:
//   fwd: xs = x + res (rounded to bf16 and stored when res != null), y = xs * rstd * w,
//        rstd = 1/sqrt(mean(xs^2) + eps)
//   bwd: g = (dy + dy2 + dy3) * w (absent terms skipped),
//        dx = rstd * (g - xs * rstd^2 * mean(g * xs)) + resid
// so a decoder block's residual adds and gradient sums cost no extra pass.
constexpr int kNormThreads = 256;

__device__ __forceinline__ void load_sum(const uint4* x, const uint4* res, long long c, float (&f)[8]) {
  bf16x8_to_f32(x[c], f);
  if (res) {
    float r[8];
    bf16x8_to_f32(res[c], r);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(__float2bfloat16_rn(f[i] + r[i]));
  }
}

__global__ void __launch_bounds__(kNormThreads) mux_rmsnorm_fwd_kernel(int dim, const uint4* x, long long ldx,
                                                                      const uint4* res, long long ldr,
                                                                      uint4* xs_out, long long ldxs, const uint4* w,
                                                                      float eps, uint4* y, long long ldy) {
  __shared__ float red[kNormThreads / 32];
  griddep_wait();
  griddep_launch_dependents();
  const long long row = blockIdx.x;
  const uint4* xr = x + row * ldx;
  const uint4* rr = res ? res + row * ldr : nullptr;
  const int nc = dim / 8;
  float ss = 0.f;
  for (int c = threadIdx.x; c < nc; c += kNormThreads) {
    float f[8];
    load_sum(xr, rr, c, f);
    if (xs_out) xs_out[row * ldxs + c] = f32_to_bf16x8(f);
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
  }
  const float rstd = rsqrtf(block_sum<kNormThreads>(ss, red) / static_cast<float>(dim) + eps);
  uint4* yr = y + row * ldy;
  for (int c = threadIdx.x; c < nc; c += kNormThreads) {
    float f[8], g[8];
    load_sum(xr, rr, c, f);
    bf16x8_to_f32(w[c], g);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = f[i] * rstd * g[i];
    yr[c] = f32_to_bf16x8(f);
  }
}

struct NormBwdIn {
  const uint4* dy[3];  // up to three upstream gradients, summed (null = absent)
  long long lddy[3];
  const uint4* resid;  // residual-path gradient added to dx (null = none)
  long long ldr;
};

__device__ __forceinline__ void load_dy(const NormBwdIn& in, long long row, int c, float (&d)[8]) {
  bf16x8_to_f32(in.dy[0][row * in.lddy[0] + c], d);
#pragma unroll
  for (int k = 1; k < 3; ++k) {
    if (in.dy[k]) {
      float e[8];
      bf16x8_to_f32(in.dy[k][row * in.lddy[k] + c], e);
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] += e[i];
    }
  }
}

__global__ void __launch_bounds__(kNormThreads) mux_rmsnorm_bwd_kernel(int dim, NormBwdIn in, const uint4* x,
                                                                      long long ldx, const uint4* w, float eps,
                                                                      uint4* dx, long long lddx) {
  __shared__ float red[kNormThreads / 32];
  griddep_wait();
  griddep_launch_dependents();
  const long long row = blockIdx.x;
  const uint4* xr = x + row * ldx;
  const int nc = dim / 8;
  float ss = 0.f, gx = 0.f;
  for (int c = threadIdx.x; c < nc; c += kNormThreads) {
    float f[8], d[8], g[8];
    bf16x8_to_f32(xr[c], f);
    load_dy(in, row, c, d);
    bf16x8_to_f32(w[c], g);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      ss = fmaf(f[i], f[i], ss);
      gx = fmaf(d[i] * g[i], f[i], gx);
    }
  }
  const float inv_dim = 1.f / static_cast<float>(dim);
  const float rstd = rsqrtf(block_sum<kNormThreads>(ss, red) * inv_dim + eps);
  const float coef = rstd * rstd * block_sum<kNormThreads>(gx, red) * inv_dim;
  uint4* dxr = dx + row * lddx;
  for (int c = threadIdx.x; c < nc; c += kNormThreads) {
    float f[8], d[8], g[8];
    bf16x8_to_f32(xr[c], f);
    load_dy(in, row, c, d);
    bf16x8_to_f32(w[c], g);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = rstd * (d[i] * g[i] - f[i] * coef);
    if (in.resid) {
      float r[8];
      bf16x8_to_f32(in.resid[row * in.ldr + c], r);
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] += r[i];
    }
    dxr[c] = f32_to_bf16x8(f);
  }
}

// ------------------------------------------------------------------ SwiGLU
__device__ __forceinline__ float sigmoidf_(float z) { return 1.f / (1.f + __expf(-z)); }

// Elementwise kernels: blocks stride over rows, threads over 16-byte column
// chunks, two chunks per thread per step so each thread has 2 x (inputs)
// loads in flight (no 64-bit index division in the loop).
#define MUX_ROWWISE_LOOP(body)                                                       \
  const int nc = dim / 8;                                                            \
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {                               \
    for (int c0 = threadIdx.x; c0 < nc; c0 += 2 * blockDim.x) {                      \
      const int c1 = c0 + blockDim.x;                                                \
      body(c0, c1 < nc, c1)                                                          \
    }                                                                                \
  }

__global__ void __launch_bounds__(256) mux_swiglu_fwd_kernel(int rows, int dim, const uint4* __restrict__ g,
                                                            long long ldg, const uint4* __restrict__ u,
                                                            long long ldu, uint4* __restrict__ h, long long ldh) {
  griddep_wait();
  griddep_launch_dependents();
#define SWIGLU_FWD(c0, two, c1)                                                       \
  const uint4 g0 = g[r * ldg + c0], u0 = u[r * ldu + c0];                             \
  uint4 g1 = make_uint4(0, 0, 0, 0), u1 = g1;                                          \
  if (two) { g1 = g[r * ldg + c1]; u1 = u[r * ldu + c1]; }                             \
  float a[8], b[8];                                                                    \
  bf16x8_to_f32(g0, a);                                                                \
  bf16x8_to_f32(u0, b);                                                                \
  _Pragma("unroll") for (int k = 0; k < 8; ++k) a[k] = a[k] * sigmoidf_(a[k]) * b[k];  \
  h[r * ldh + c0] = f32_to_bf16x8(a);                                                  \
  if (two) {                                                                           \
    bf16x8_to_f32(g1, a);                                                              \
    bf16x8_to_f32(u1, b);                                                              \
    _Pragma("unroll") for (int k = 0; k < 8; ++k) a[k] = a[k] * sigmoidf_(a[k]) * b[k];\
    h[r * ldh + c1] = f32_to_bf16x8(a);                                                \
  }
  MUX_ROWWISE_LOOP(SWIGLU_FWD)
#undef SWIGLU_FWD
}

// dg = dh * u * s (1 + g (1 - s)),  du = dh * g * s,  s = sigmoid(g)
__device__ __forceinline__ void swiglu_bwd8(const uint4 dh, const uint4 g, const uint4 u, uint4& dg, uint4& du) {
  float d[8], a[8], b[8], o1[8], o2[8];
  bf16x8_to_f32(dh, d);
  bf16x8_to_f32(g, a);
  bf16x8_to_f32(u, b);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float s = sigmoidf_(a[k]);
    o1[k] = d[k] * b[k] * s * (1.f + a[k] * (1.f - s));
    o2[k] = d[k] * a[k] * s;
  }
  dg = f32_to_bf16x8(o1);
  du = f32_to_bf16x8(o2);
}

__global__ void __launch_bounds__(256) mux_swiglu_bwd_kernel(int rows, int dim, const uint4* __restrict__ dh,
                                                            long long lddh, const uint4* __restrict__ g,
                                                            long long ldg, const uint4* __restrict__ u,
                                                            long long ldu, uint4* __restrict__ dg, long long lddg,
                                                            uint4* __restrict__ du, long long lddu) {
  griddep_wait();
  griddep_launch_dependents();
#define SWIGLU_BWD(c0, two, c1)                                                       \
  const uint4 d0 = dh[r * lddh + c0], g0 = g[r * ldg + c0], u0 = u[r * ldu + c0];      \
  uint4 d1 = make_uint4(0, 0, 0, 0), g1 = d1, u1 = d1;                                 \
  if (two) { d1 = dh[r * lddh + c1]; g1 = g[r * ldg + c1]; u1 = u[r * ldu + c1]; }     \
  uint4 o1, o2;                                                                        \
  swiglu_bwd8(d0, g0, u0, o1, o2);                                                     \
  dg[r * lddg + c0] = o1;                                                              \
  du[r * lddu + c0] = o2;                                                              \
  if (two) {                                                                           \
    swiglu_bwd8(d1, g1, u1, o1, o2);                                                   \
    dg[r * lddg + c1] = o1;                                                            \
    du[r * lddu + c1] = o2;                                                            \
  }
  MUX_ROWWISE_LOOP(SWIGLU_BWD)
#undef SWIGLU_BWD
}

// ------------------------------------------------------------------ residual add
__device__ __forceinline__ uint4 add8(const uint4 a, const uint4 b) {
  float x[8], z[8];
  bf16x8_to_f32(a, x);
  bf16x8_to_f32(b, z);
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] += z[k];
  return f32_to_bf16x8(x);
}

__global__ void __launch_bounds__(256) mux_add_kernel(int rows, int dim, const uint4* a, long long lda,
                                                     const uint4* b, long long ldb, uint4* y, long long ldy) {
  griddep_wait();
  griddep_launch_dependents();
#define ADD_BODY(c0, two, c1)                                                         \
  const uint4 a0 = a[r * lda + c0], b0 = b[r * ldb + c0];                              \
  uint4 a1 = make_uint4(0, 0, 0, 0), b1 = a1;                                          \
  if (two) { a1 = a[r * lda + c1]; b1 = b[r * ldb + c1]; }                             \
  y[r * ldy + c0] = add8(a0, b0);                                                      \
  if (two) y[r * ldy + c1] = add8(a1, b1);
  MUX_ROWWISE_LOOP(ADD_BODY)
#undef ADD_BODY
}

// ------------------------------------------------------------------ RoPE
// In place on x [rows, heads * d] (row stride ld): pairs (i, i + d/2) of each
// head rotated by theta_i = pos * base^(-2i/d), pos = r - row_start[r]
// (inverse != 0: by -theta, the backward).  Pad rows are left untouched.
// One thread per (row, 8 consecutive i): its 8 angles are computed once and
// applied to every head of the row.
__global__ void __launch_bounds__(256) mux_rope_kernel(int rows, int heads, int d, uint4* x, long long ld,
                                                      const int32_t* row_start, float log2_base, int inverse) {
  griddep_wait();
  griddep_launch_dependents();
  const int half_c = d / 16;  // 8-wide chunks per half head
  const long long total = static_cast<long long>(rows) * half_c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / half_c;
    const int c = static_cast<int>(i - r * half_c);
    const int rs = row_start[r];
    if (rs < 0) continue;
    const float pos = static_cast<float>(r - rs);
    float cs[8], sn[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float inv_freq = exp2f(-2.f * static_cast<float>(8 * c + k) / static_cast<float>(d) * log2_base);
      sincosf(pos * inv_freq, &sn[k], &cs[k]);
      if (inverse) sn[k] = -sn[k];
    }
    uint4* row = x + r * ld;
    for (int h = 0; h < heads; ++h) {
      uint4* base = row + (static_cast<long long>(h) * d) / 8;
      float a[8], b[8];
      bf16x8_to_f32(base[c], a);
      bf16x8_to_f32(base[c + half_c], b);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float x0 = a[k], x1 = b[k];
        a[k] = x0 * cs[k] - x1 * sn[k];
        b[k] = x1 * cs[k] + x0 * sn[k];
      }
      base[c] = f32_to_bf16x8(a);
      base[c + half_c] = f32_to_bf16x8(b);
    }
  }
}

// ------------------------------------------------------------------ launchers
// row-strided elementwise kernels: 8 resident 256-thread blocks per SM
static unsigned grid_rows(int rows, int num_sms) {
  const int cap = num_sms * 8;
  return static_cast<unsigned>(rows < 1 ? 1 : (rows < cap ? rows : cap));
}

static unsigned grid_for(long long work, int per_block, int num_sms) {
  long long b = (work + per_block - 1) / per_block;
  const long long cap = static_cast<long long>(num_sms) * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

cudaError_t launch_row_start(int num_seqs, const int32_t* seq_len, const int32_t* seq_row, int max_rows,
                             int32_t* row_start, int num_sms, cudaStream_t s) {
  cudaError_t e = launch_pdl(mux_row_fill_kernel, dim3(grid_for(max_rows, 256, num_sms)), dim3(256), 0, s,
                             row_start, max_rows);
  if (e != cudaSuccess || num_seqs == 0) return e;
  return launch_pdl(mux_row_scatter_kernel, dim3(std::min(num_seqs, num_sms * 8)), dim3(256), 0, s, num_seqs,
                    seq_len, seq_row, row_start, max_rows);
}

cudaError_t launch_rmsnorm_fwd(int rows, int dim, const void* x, long long ldx, const void* res, long long ldr,
                               void* xs, long long ldxs, const void* w, float eps, void* y, long long ldy,
                               cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  return launch_pdl(mux_rmsnorm_fwd_kernel, dim3(rows), dim3(kNormThreads), 0, s, dim, static_cast<const uint4*>(x),
                    ldx / 8, static_cast<const uint4*>(res), ldr / 8, static_cast<uint4*>(xs), ldxs / 8,
                    static_cast<const uint4*>(w), eps, static_cast<uint4*>(y), ldy / 8);
}

cudaError_t launch_rmsnorm_bwd(int rows, int dim, const void* const* dy, const long long* lddy, const void* resid,
                               long long ldr, const void* x, long long ldx, const void* w, float eps, void* dx,
                               long long lddx, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  NormBwdIn in;
  for (int k = 0; k < 3; ++k) {
    in.dy[k] = static_cast<const uint4*>(dy[k]);
    in.lddy[k] = lddy[k] / 8;
  }
  in.resid = static_cast<const uint4*>(resid);
  in.ldr = ldr / 8;
  return launch_pdl(mux_rmsnorm_bwd_kernel, dim3(rows), dim3(kNormThreads), 0, s, dim, in,
                    static_cast<const uint4*>(x), ldx / 8, static_cast<const uint4*>(w), eps, static_cast<uint4*>(dx),
                    lddx / 8);
}

cudaError_t launch_swiglu_fwd(int rows, int dim, const void* g, long long ldg, const void* u, long long ldu, void* h,
                              long long ldh, int num_sms, cudaStream_t s) {
  const long long work = static_cast<long long>(rows) * (dim / 8);
  if (work == 0) return cudaSuccess;
  return launch_pdl(mux_swiglu_fwd_kernel, dim3(grid_rows(rows, num_sms)), dim3(256), 0, s, rows, dim,
                    static_cast<const uint4*>(g), ldg / 8, static_cast<const uint4*>(u), ldu / 8,
                    static_cast<uint4*>(h), ldh / 8);
}

cudaError_t launch_swiglu_bwd(int rows, int dim, const void* dh, long long lddh, const void* g, long long ldg,
                              const void* u, long long ldu, void* dg, long long lddg, void* du, long long lddu,
                              int num_sms, cudaStream_t s) {
  const long long work = static_cast<long long>(rows) * (dim / 8);
  if (work == 0) return cudaSuccess;
  return launch_pdl(mux_swiglu_bwd_kernel, dim3(grid_rows(rows, num_sms)), dim3(256), 0, s, rows, dim,
                    static_cast<const uint4*>(dh), lddh / 8, static_cast<const uint4*>(g), ldg / 8,
                    static_cast<const uint4*>(u), ldu / 8, static_cast<uint4*>(dg), lddg / 8,
                    static_cast<uint4*>(du), lddu / 8);
}

cudaError_t launch_add(int rows, int dim, const void* a, long long lda, const void* b, long long ldb, void* y,
                       long long ldy, int num_sms, cudaStream_t s) {
  const long long work = static_cast<long long>(rows) * (dim / 8);
  if (work == 0) return cudaSuccess;
  return launch_pdl(mux_add_kernel, dim3(grid_rows(rows, num_sms)), dim3(256), 0, s, rows, dim,
                    static_cast<const uint4*>(a), lda / 8, static_cast<const uint4*>(b), ldb / 8,
                    static_cast<uint4*>(y), ldy / 8);
}

cudaError_t launch_rope(int rows, int heads, int d, void* x, long long ld, const int32_t* row_start, float base,
                        bool inverse, int num_sms, cudaStream_t s) {
  const long long work = static_cast<long long>(rows) * (d / 16);
  if (work == 0 || heads == 0) return cudaSuccess;
  return launch_pdl(mux_rope_kernel, dim3(grid_for(work, 256, num_sms)), dim3(256), 0, s, rows, heads, d,
                    static_cast<uint4*>(x), ld / 8, row_start, log2f(base), inverse ? 1 : 0);
}

}  // namespace mux
