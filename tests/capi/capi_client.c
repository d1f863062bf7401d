/* A plain-C client of the drop-in boundary (include/rbc.h): what a maintainer
 * binding librbc.so from C (or cgo / JNI / FFI) would write.
 *
 *   gcc -std=c99 -I include tests/capi/capi_client.c -L paper_1905_07439_b200/lib -lrbc -lm
 *
 * 1. rbc_leaf_matmul (reference _engine.py:42-61): the exact-order product of
 *    two binary64 matrices equals the same k-ascending loop in C bit for bit.
 * 2. rbc_apply_levels (reference _engine.py:117-149) with Strassen's tensors
 *    at Q = 2: equals the C restatement of the breadth-first recursion below
 *    (rounded multiply and add kept separate: compile without FMA contraction)
 *    bit for bit; an indivisible size returns RBC_EVALUE with a message.
 * Exit code 0 on success; prints the failing check otherwise. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rbc.h"

#define N 8
#define R 7

/* Strassen <2,2,2;7>, the reference's constants (formula.py:98-114): u[r][k][l] */
static const double SU[R][2][2] = {{{1, 0}, {0, 1}}, {{0, 0}, {1, 1}}, {{1, 0}, {0, 0}}, {{0, 0}, {0, 1}},
                                   {{1, 1}, {0, 0}}, {{-1, 0}, {1, 0}}, {{0, 1}, {0, -1}}};
static const double SV[R][2][2] = {{{1, 0}, {0, 1}}, {{1, 0}, {0, 0}}, {{0, 1}, {0, -1}}, {{-1, 0}, {1, 0}},
                                   {{0, 0}, {0, 1}}, {{1, 1}, {0, 0}}, {{0, 0}, {1, 1}}};
static const double SW[R][2][2] = {{{1, 0}, {0, 1}}, {{0, 0}, {1, -1}}, {{0, 1}, {0, 1}}, {{1, 0}, {1, 0}},
                                   {{-1, 1}, {0, 0}}, {{0, 0}, {0, 1}}, {{1, 0}, {0, 0}}};

static volatile double sink; /* keeps the compiler from contracting mul + add */
static double mul(double a, double b) { double p = a * b; sink = p; return p; }
static double add(double a, double b) { double s = a + b; sink = s; return s; }

/* reference recursion on an s x s block (row stride ld), depth q levels left */
static void bc(const double* x, const double* y, double* out, int s, int ld, int q) {
  if (q == 0) { /* leaf: k ascending, first term initialises */
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        double acc = mul(x[i * ld], y[j]);
        for (int k = 1; k < s; ++k) acc = add(acc, mul(x[i * ld + k], y[k * ld + j]));
        out[i * ld + j] = acc;
      }
    return;
  }
  const int h = s / 2;
  double* xs = malloc(sizeof(double) * h * h);
  double* ys = malloc(sizeof(double) * h * h);
  double* ps = malloc(sizeof(double) * R * h * h);
  for (int r = 0; r < R; ++r) {
    for (int i = 0; i < h; ++i)
      for (int j = 0; j < h; ++j) { /* row sums folded left, then the rows */
        double ex = 0, ey = 0;
        for (int k = 0; k < 2; ++k) {
          double rx = mul(SU[r][k][0], x[(k * h + i) * ld + j]);
          rx = add(rx, mul(SU[r][k][1], x[(k * h + i) * ld + h + j]));
          double ry = mul(SV[r][k][0], y[(k * h + i) * ld + j]);
          ry = add(ry, mul(SV[r][k][1], y[(k * h + i) * ld + h + j]));
          ex = k == 0 ? rx : add(ex, rx);
          ey = k == 0 ? ry : add(ey, ry);
        }
        xs[i * h + j] = ex;
        ys[i * h + j] = ey;
      }
    bc(xs, ys, ps + r * h * h, h, h, q - 1);
  }
  for (int I = 0; I < 2; ++I)
    for (int J = 0; J < 2; ++J)
      for (int i = 0; i < h; ++i)
        for (int j = 0; j < h; ++j) { /* fold over r ascending, first term initialises */
          double acc = mul(SW[0][I][J], ps[i * h + j]);
          for (int r = 1; r < R; ++r) acc = add(acc, mul(SW[r][I][J], ps[r * h * h + i * h + j]));
          out[(I * h + i) * ld + J * h + j] = acc;
        }
  free(xs); free(ys); free(ps);
}

static int same_values(const double* a, const double* b, int n) {
  for (int i = 0; i < n; ++i)
    if (!(a[i] == b[i])) return 0; /* np.array_equal: the sign of a zero may differ */
  return 1;
}

int main(void) {
  if (rbc_abi_version() != RBC_ABI_VERSION) { puts("ABI version mismatch"); return 1; }
  if (rbc_device_count() < 1) { puts("no CUDA device"); return 2; }
  double a[N * N], b[N * N], got[N * N], want[N * N];
  unsigned s = 12345u;
  for (int i = 0; i < N * N; ++i) {
    s = s * 1664525u + 1013904223u; a[i] = (double)(s >> 8) / 16777216.0 - 0.5;
    s = s * 1664525u + 1013904223u; b[i] = (double)(s >> 8) / 16777216.0 - 0.5;
  }
  /* 1. leaf */
  if (rbc_leaf_matmul(RBC_F64, 1, N * N, N * N, N, N, N, a, b, got) != RBC_OK) {
    printf("rbc_leaf_matmul: %s\n", rbc_last_error()); return 3;
  }
  bc(a, b, want, N, N, 0);
  if (memcmp(got, want, sizeof got) != 0) { puts("leaf differs from the C loop"); return 4; }
  /* 2. two Strassen levels */
  const int32_t nn[2] = {2, 2}, rr[2] = {R, R};
  const int64_t tc[2] = {1, 1};
  const void* u[2] = {SU, SU};
  const void* v[2] = {SV, SV};
  const void* w[2] = {SW, SW};
  uint64_t leaves = 0;
  if (rbc_apply_levels(RBC_F64, 2, nn, rr, tc, u, v, w, 1, N, a, b, 1, got, &leaves) != RBC_OK) {
    printf("rbc_apply_levels: %s\n", rbc_last_error()); return 5;
  }
  bc(a, b, want, N, N, 2);
  if (!same_values(got, want, N * N)) { puts("apply_levels differs from the C recursion"); return 6; }
  if (leaves != 49) { printf("leaf count %llu, want 49\n", (unsigned long long)leaves); return 7; }
  /* 3. error mapping: 6 is not divisible by 2 twice */
  double a6[36] = {0}, o6[36];
  const int rc = rbc_apply_levels(RBC_F64, 2, nn, rr, tc, u, v, w, 1, 6, a6, a6, 1, o6, &leaves);
  if (rc != RBC_EVALUE || strstr(rbc_last_error(), "divisible") == NULL) {
    printf("indivisible size: rc %d, message '%s'\n", rc, rbc_last_error()); return 8;
  }
  puts("capi client ok");
  return 0;
}
