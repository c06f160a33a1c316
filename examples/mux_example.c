/* mux_example.c — the C ABI used directly from C (no Python, no torch).
 *
 * Packs two tasks' sequences (mux_pack_chunks), gathers their token rows into
 * the packed layout (mux_pack_apply), runs the fused multiplexed LoRA linear
 * forward and backward (mux_linear_fwd / mux_linear_bwd) and prints a few
 * values.  Build (see tests/test_c_example.py):
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/mux_example.c \
 *       -L paper_2603_02885_b200 -l:libmux.so -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2603_02885_b200 -o build/mux_example
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "mux.h"

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 2;                                                               \
    }                                                                         \
  } while (0)
#define MK(x)                                                                 \
  do {                                                                        \
    mux_status s_ = (x);                                                      \
    if (s_ != MUX_OK) {                                                       \
      fprintf(stderr, "%s:%d mux status %d: %s\n", __FILE__, __LINE__, (int)s_, mux_last_error()); \
      return 3;                                                               \
    }                                                                         \
  } while (0)

static unsigned short f2bf(float f) { /* round to nearest even */
  unsigned int u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (unsigned short)(u >> 16);
}
static float bf2f(unsigned short b) {
  unsigned int u = (unsigned int)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static float frand(unsigned int* s) { /* xorshift in [-1, 1) */
  *s ^= *s << 13; *s ^= *s >> 17; *s ^= *s << 5;
  return (float)(*s & 0xFFFFFF) / (float)0x800000 - 1.0f;
}

int main(void) {
  printf("%s\n", mux_version());
  const int M = 2, S = 3, K = 256, N = 256, R_CAP = 16;
  const int task_seq_off[3] = {0, 2, 3};
  const int seq_len[3] = {100, 20, 64}; /* task 0: 100 + 20, task 1: 64 */
  const int T = 184;
  const int max_rows = (int)mux_pack_bound_rows(T, S, 64);
  const int max_chunks = max_rows / 64;

  int *d_off, *d_len, *d_seg, *d_seq_row, *d_ct, *d_cp, *d_cv, *d_cd, *d_rs;
  mux_pack_info* d_info;
  void* d_pws;
  size_t pws = mux_pack_workspace_size(M, S);
  CK(cudaMalloc((void**)&d_off, sizeof(task_seq_off)));
  CK(cudaMalloc((void**)&d_len, sizeof(seq_len)));
  CK(cudaMalloc((void**)&d_seg, (M + 1) * sizeof(int)));
  CK(cudaMalloc((void**)&d_seq_row, S * sizeof(int)));
  CK(cudaMalloc((void**)&d_ct, max_chunks * sizeof(int)));
  CK(cudaMalloc((void**)&d_cp, max_chunks * sizeof(int)));
  CK(cudaMalloc((void**)&d_cv, max_chunks * sizeof(int)));
  CK(cudaMalloc((void**)&d_cd, max_chunks * sizeof(int)));
  CK(cudaMalloc((void**)&d_rs, max_rows * sizeof(int)));
  CK(cudaMalloc((void**)&d_info, sizeof(mux_pack_info)));
  CK(cudaMalloc(&d_pws, pws));
  CK(cudaMemcpy(d_off, task_seq_off, sizeof(task_seq_off), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_len, seq_len, sizeof(seq_len), cudaMemcpyHostToDevice));
  MK(mux_pack_chunks(M, S, d_off, d_len, NULL, 0, 64, max_rows, max_chunks, d_seg, d_seq_row, d_ct, d_cp, d_cv,
                     d_cd, d_rs, d_info, d_pws, pws, 0));
  mux_pack_info info;
  int seg_off[3];
  CK(cudaMemcpy(&info, d_info, sizeof(info), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(seg_off, d_seg, sizeof(seg_off), cudaMemcpyDeviceToHost));
  printf("pack: chunk %d, chunks %d, rows %d (valid %d), seg_off = [%d %d %d]\n", info.chunk_size, info.num_chunks,
         info.total_rows, info.valid_rows, seg_off[0], seg_off[1], seg_off[2]);

  /* host data */
  unsigned int seed = 12345u;
  unsigned short* hX = malloc(sizeof(unsigned short) * T * K);
  unsigned short* hW = malloc(sizeof(unsigned short) * N * K);
  unsigned short* hdY = malloc(sizeof(unsigned short) * max_rows * N);
  for (int i = 0; i < T * K; ++i) hX[i] = f2bf(frand(&seed));
  for (int i = 0; i < N * K; ++i) hW[i] = f2bf(frand(&seed) / 16.0f);
  for (int i = 0; i < max_rows * N; ++i) hdY[i] = f2bf(frand(&seed));
  const int ranks[2] = {16, 8};
  const int ldb[2] = {16, 8};
  unsigned short *hA[2], *hB[2];
  for (int t = 0; t < 2; ++t) {
    hA[t] = malloc(sizeof(unsigned short) * ranks[t] * K);
    hB[t] = malloc(sizeof(unsigned short) * N * ldb[t]);
    for (int i = 0; i < ranks[t] * K; ++i) hA[t][i] = f2bf(frand(&seed) / 16.0f);
    for (int i = 0; i < N * ldb[t]; ++i) hB[t][i] = f2bf(frand(&seed));
  }
  mux_bf16 *dXtok, *dX, *dW, *dY, *dHs, *ddY, *ddX, *dA[2], *dB[2];
  float *gA[2], *gB[2];
  CK(cudaMalloc((void**)&dXtok, sizeof(short) * T * K));
  CK(cudaMalloc((void**)&dX, sizeof(short) * max_rows * K));
  CK(cudaMalloc((void**)&dW, sizeof(short) * N * K));
  CK(cudaMalloc((void**)&dY, sizeof(short) * max_rows * N));
  CK(cudaMalloc((void**)&dHs, sizeof(short) * max_rows * R_CAP));
  CK(cudaMalloc((void**)&ddY, sizeof(short) * max_rows * N));
  CK(cudaMalloc((void**)&ddX, sizeof(short) * max_rows * K));
  CK(cudaMemcpy(dXtok, hX, sizeof(short) * T * K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dW, hW, sizeof(short) * N * K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ddY, hdY, sizeof(short) * max_rows * N, cudaMemcpyHostToDevice));
  mux_adapter ad[2];
  for (int t = 0; t < 2; ++t) {
    CK(cudaMalloc((void**)&dA[t], sizeof(short) * ranks[t] * K));
    CK(cudaMalloc((void**)&dB[t], sizeof(short) * N * ldb[t]));
    CK(cudaMalloc((void**)&gA[t], sizeof(float) * ranks[t] * K));
    CK(cudaMalloc((void**)&gB[t], sizeof(float) * N * ranks[t]));
    CK(cudaMemcpy(dA[t], hA[t], sizeof(short) * ranks[t] * K, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB[t], hB[t], sizeof(short) * N * ldb[t], cudaMemcpyHostToDevice));
    ad[t].A = dA[t];
    ad[t].B = dB[t];
    ad[t].dA = gA[t];
    ad[t].dB = gB[t];
    ad[t].rank = ranks[t];
    ad[t].ldb = ldb[t];
    ad[t].scale = 2.0f;
  }
  const int seg_task[2] = {0, 1};
  size_t wsb = mux_linear_workspace_size(2, max_rows, K, N, R_CAP);
  void* ws;
  CK(cudaMalloc(&ws, wsb));
  CK(cudaMemset(ws, 0, wsb)); /* zero once; reusable afterwards */

  MK(mux_pack_apply(max_rows, K, T, d_rs, dXtok, dX, 0));
  MK(mux_linear_fwd(2, d_seg, seg_task, 2, ad, max_rows, K, N, R_CAP, dX, dW, dY, dHs, ws, wsb, 0));
  MK(mux_linear_bwd(2, d_seg, seg_task, 2, ad, max_rows, K, N, R_CAP, ddY, dX, dW, dHs, ddX, ws, wsb, 0));
  CK(cudaDeviceSynchronize());

  unsigned short y[4];
  float ga[2];
  CK(cudaMemcpy(y, dY, sizeof(y), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ga, gA[0], sizeof(ga), cudaMemcpyDeviceToHost));
  printf("Y[0,0:4] = %.4f %.4f %.4f %.4f   dA_0[0,0:2] = %.4f %.4f\n", bf2f(y[0]), bf2f(y[1]), bf2f(y[2]),
         bf2f(y[3]), ga[0], ga[1]);
  /* a fused projection through the generic entry point: W2 = [W; W] (512 output columns in two
   * slices), each task with one adapter per slice (slice 0: the adapters above, slice 1: the same A
   * with scale 1); slice 0 of the output must equal the plain call's Y bit for bit. */
  {
    mux_bf16 *dW2, *dY2, *dHs2;
    CK(cudaMalloc((void**)&dW2, sizeof(short) * 2 * N * K));
    CK(cudaMalloc((void**)&dY2, sizeof(short) * max_rows * 2 * N));
    CK(cudaMalloc((void**)&dHs2, sizeof(short) * max_rows * 2 * R_CAP));
    CK(cudaMemcpy(dW2, dW, sizeof(short) * N * K, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(dW2 + (size_t)N * K, dW, sizeof(short) * N * K, cudaMemcpyDeviceToDevice));
    mux_adapter ad2[4];
    for (int t = 0; t < 2; ++t) {
      ad2[2 * t] = ad[t];
      ad2[2 * t + 1] = ad[t];
      ad2[2 * t + 1].scale = 1.0f;
    }
    mux_slices sl = {2, {0, N, 2 * N, 0, 0}};
    size_t wsb2 = mux_linear_workspace_size(2, max_rows, K, 2 * N, 2 * R_CAP);
    void* ws2;
    CK(cudaMalloc(&ws2, wsb2));
    CK(cudaMemset(ws2, 0, wsb2));
    mux_linear_args a;
    memset(&a, 0, sizeof(a));
    a.op = MUX_OP_FWD;
    a.num_segs = 2;
    a.seg_off = d_seg;
    a.seg_task = seg_task;
    a.num_adapters = 2;
    a.adapters = ad2;
    a.slices = &sl;
    a.max_rows = max_rows;
    a.K = K;
    a.N = 2 * N;
    a.r_cap = R_CAP;
    a.X = dX;
    a.W = dW2;
    a.Y = dY2;
    a.Hs = dHs2;
    a.workspace = ws2;
    a.workspace_bytes = wsb2;
    MK(mux_linear(&a));
    CK(cudaDeviceSynchronize());
    unsigned short* y1 = malloc(sizeof(short) * info.total_rows * N);
    unsigned short* y2 = malloc(sizeof(short) * info.total_rows * 2 * N);
    CK(cudaMemcpy(y1, dY, sizeof(short) * info.total_rows * N, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y2, dY2, sizeof(short) * info.total_rows * 2 * N, cudaMemcpyDeviceToHost));
    int same = 1;
    for (int r = 0; r < info.total_rows; ++r)
      for (int c = 0; c < N; ++c) same &= y1[(size_t)r * N + c] == y2[(size_t)r * 2 * N + c];
    printf("sliced: slice 0 == plain Y: %s\n", same ? "yes" : "no");
    free(y1);
    free(y2);
  }
  /* an invalid call: K not a multiple of 8 -> MUX_ERR_INVALID_ARGUMENT, nothing launched */
  mux_status bad = mux_linear_fwd(2, d_seg, seg_task, 2, ad, max_rows, 100, N, R_CAP, dX, dW, dY, dHs, ws, wsb, 0);
  printf("invalid K -> status %d (%s)\n", (int)bad, mux_last_error());
  printf("ok\n");
  return 0;
}
