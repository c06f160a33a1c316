/* fp64 CPU ORACLE for the multiplexed LoRA linear — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code with the CUDA path.
 *
 * What it computes (definitions, not an algorithm):
 *   Paper Eq. 1 (§3.2 "BaseOp fwd"):  [X_1;X_2] W = [X_1 W; X_2 W]
 *   Paper Eq. 2 (§3.2 "BaseOp bwd"):  G^in = [G^out_1;G^out_2] W^T
 *   LoRA per task (north_star; the paper cites LoRA at P:244/P:456 without a
 *   formula — reading Q1/Q2 in DESIGN.md): with W [N,K], A_t [r_t,K],
 *   B_t [N,r_t] (nn.Linear / PEFT layouts), for every row i of segment s
 *   (seg_off[s] <= i < seg_off[s+1]) owned by adapter t = seg_task[s]:
 *     H[i,j]  = sum_k X[i,k] A_t[j,k]                          (j < r_t)
 *     Y[i,n]  = sum_k X[i,k] W[n,k] + s_t * sum_j H[i,j] B_t[n,j]
 *     Hs[i,j] = s_t * H[i,j]   (j < r_t),  0 for r_t <= j < r_cap
 *   backward (chain rule of the above; no backbone dW):
 *     G[i,j]  = sum_n dY[i,n] B_t[n,j]
 *     dX[i,k] = sum_n dY[i,n] W[n,k] + s_t * sum_j G[i,j] A_t[j,k]
 *     dA_t[j,k] = s_t * sum_{i in segs of t} G[i,j] X[i,k]
 *     dB_t[n,j] = s_t * sum_{i in segs of t} dY[i,n] H[i,j]
 *     Gs[i,j] = s_t * G[i,j]
 * Every sum runs in ascending index order in fp64; OpenMP only splits
 * independent output elements, so results are bitwise deterministic and a
 * row's result does not depend on which other rows/tasks are present.
 * Rows outside every segment are not computed (outputs left untouched).
 * Y / dX can be restricted to a row sample (rows[], num_rows; NULL = all rows
 * of all segments, outputs then indexed by row); H, G, dA, dB always use all
 * rows.  Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC.
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>

typedef struct {
  const double* A;   /* [rank, K] */
  const double* B;   /* [N, rank] */
  double* dA;        /* [rank, K] out (bwd), may be NULL */
  double* dB;        /* [N, rank] out (bwd), may be NULL */
  int32_t rank;
  double scale;
} oracle_adapter;

static int seg_of_row(int num_segs, const int32_t* seg_off, int64_t i) {
  for (int s = 0; s < num_segs; ++s)
    if (seg_off[s] <= i && i < seg_off[s + 1]) return s;
  return -1;
}

/* H (unscaled) for every row of every segment: H[i*r_cap + j]. */
static void compute_H(int num_segs, const int32_t* seg_off, const int32_t* seg_task,
                      const oracle_adapter* ad, int64_t K, int r_cap,
                      const double* X, double* H) {
  int64_t R = seg_off[num_segs];
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < R; ++i) {
    int s = seg_of_row(num_segs, seg_off, i);
    for (int j = 0; j < r_cap; ++j) H[i * r_cap + j] = 0.0;
    if (s < 0) continue;
    const oracle_adapter* a = &ad[seg_task[s]];
    for (int j = 0; j < a->rank; ++j) {
      double acc = 0.0;
      for (int64_t k = 0; k < K; ++k) acc += X[i * K + k] * a->A[(int64_t)j * K + k];
      H[i * r_cap + j] = acc;
    }
  }
}

/* G (unscaled): G[i,j] = sum_n dY[i,n] B_t[n,j]. */
static void compute_G(int num_segs, const int32_t* seg_off, const int32_t* seg_task,
                      const oracle_adapter* ad, int64_t N, int r_cap,
                      const double* dY, double* G) {
  int64_t R = seg_off[num_segs];
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < R; ++i) {
    int s = seg_of_row(num_segs, seg_off, i);
    for (int j = 0; j < r_cap; ++j) G[i * r_cap + j] = 0.0;
    if (s < 0) continue;
    const oracle_adapter* a = &ad[seg_task[s]];
    for (int j = 0; j < a->rank; ++j) {
      double acc = 0.0;
      for (int64_t n = 0; n < N; ++n) acc += dY[i * N + n] * a->B[n * a->rank + j];
      G[i * r_cap + j] = acc;
    }
  }
}

/* Forward.  X [R,K], W [N,K]; outputs Y [num_rows or R, N], Hs [R, r_cap]. */
int oracle_linear_fwd(int num_segs, const int32_t* seg_off, const int32_t* seg_task,
                      int num_adapters, const oracle_adapter* ad,
                      int64_t K, int64_t N, int r_cap,
                      const double* X, const double* W,
                      const int64_t* rows, int64_t num_rows,
                      double* Y, double* Hs) {
  (void)num_adapters;
  int64_t R = seg_off[num_segs];
  double* H = (double*)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1) * (size_t)(r_cap > 0 ? r_cap : 1));
  if (!H) return 1;
  compute_H(num_segs, seg_off, seg_task, ad, K, r_cap, X, H);
  if (Hs) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < R; ++i) {
      int s = seg_of_row(num_segs, seg_off, i);
      double sc = s >= 0 ? ad[seg_task[s]].scale : 0.0;
      for (int j = 0; j < r_cap; ++j) Hs[i * r_cap + j] = sc * H[i * r_cap + j];
    }
  }
  if (Y) {
    int64_t nr = rows ? num_rows : R;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nr; ++q) {
      int64_t i = rows ? rows[q] : q;
      int s = seg_of_row(num_segs, seg_off, i);
      if (s < 0) continue;
      const oracle_adapter* a = &ad[seg_task[s]];
      for (int64_t n = 0; n < N; ++n) {
        double base = 0.0;
        for (int64_t k = 0; k < K; ++k) base += X[i * K + k] * W[n * K + k];
        double lora = 0.0;
        for (int j = 0; j < a->rank; ++j) lora += H[i * r_cap + j] * a->B[n * a->rank + j];
        Y[q * N + n] = base + a->scale * lora;
      }
    }
  }
  free(H);
  return 0;
}

/* Backward.  dY [R,N], X [R,K], W [N,K]; outputs dX [num_rows or R, K],
 * Gs [R, r_cap] (may be NULL), dA/dB through the adapter table. */
int oracle_linear_bwd(int num_segs, const int32_t* seg_off, const int32_t* seg_task,
                      int num_adapters, const oracle_adapter* ad,
                      int64_t K, int64_t N, int r_cap,
                      const double* dY, const double* X, const double* W,
                      const int64_t* rows, int64_t num_rows,
                      double* dX, double* Gs) {
  int64_t R = seg_off[num_segs];
  size_t hsz = sizeof(double) * (size_t)(R > 0 ? R : 1) * (size_t)(r_cap > 0 ? r_cap : 1);
  double* H = (double*)malloc(hsz);
  double* G = (double*)malloc(hsz);
  if (!H || !G) { free(H); free(G); return 1; }
  compute_H(num_segs, seg_off, seg_task, ad, K, r_cap, X, H);
  compute_G(num_segs, seg_off, seg_task, ad, N, r_cap, dY, G);
  if (Gs) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < R; ++i) {
      int s = seg_of_row(num_segs, seg_off, i);
      double sc = s >= 0 ? ad[seg_task[s]].scale : 0.0;
      for (int j = 0; j < r_cap; ++j) Gs[i * r_cap + j] = sc * G[i * r_cap + j];
    }
  }
  if (dX) {
    int64_t nr = rows ? num_rows : R;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nr; ++q) {
      int64_t i = rows ? rows[q] : q;
      int s = seg_of_row(num_segs, seg_off, i);
      if (s < 0) continue;
      const oracle_adapter* a = &ad[seg_task[s]];
      for (int64_t k = 0; k < K; ++k) {
        double base = 0.0;
        for (int64_t n = 0; n < N; ++n) base += dY[i * N + n] * W[n * K + k];
        double lora = 0.0;
        for (int j = 0; j < a->rank; ++j) lora += G[i * r_cap + j] * a->A[(int64_t)j * K + k];
        dX[q * K + k] = base + a->scale * lora;
      }
    }
  }
  /* adapter gradients: sum over every segment owned by the adapter, rows ascending */
  for (int t = 0; t < num_adapters; ++t) {
    const oracle_adapter* a = &ad[t];
    int r = a->rank;
    if (a->dA) {
      #pragma omp parallel for schedule(static)
      for (int64_t k = 0; k < K; ++k) {
        for (int j = 0; j < r; ++j) {
          double acc = 0.0;
          for (int s = 0; s < num_segs; ++s) {
            if (seg_task[s] != t) continue;
            for (int64_t i = seg_off[s]; i < seg_off[s + 1]; ++i)
              acc += G[i * r_cap + j] * X[i * K + k];
          }
          a->dA[(int64_t)j * K + k] = a->scale * acc;
        }
      }
    }
    if (a->dB) {
      #pragma omp parallel for schedule(static)
      for (int64_t n = 0; n < N; ++n) {
        for (int j = 0; j < r; ++j) {
          double acc = 0.0;
          for (int s = 0; s < num_segs; ++s) {
            if (seg_task[s] != t) continue;
            for (int64_t i = seg_off[s]; i < seg_off[s + 1]; ++i)
              acc += dY[i * N + n] * H[i * r_cap + j];
          }
          a->dB[n * r + j] = a->scale * acc;
        }
      }
    }
  }
  free(H);
  free(G);
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* thread count of the OpenMP loops (timing only: the result does not depend on it) */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}
