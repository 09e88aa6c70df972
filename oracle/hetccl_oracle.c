/*
 * hetccl_oracle.c — plain, slow, obviously-correct CPU oracle for the hierarchical collectives.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this. It includes no CUDA header and shares no code with
 * paper_2601_22585_b200/ (the product path); neither side imports the other.
 *
 * What it computes:
 *   The collectives the paper evaluates — All-Reduce, Reduce-Scatter, All-Gather, Broadcast
 *   (§5.2 "All-Reduce, All-Gather, Reduce-Scatter, Reduce, Broadcast, and All-to-All";
 *   PAPER.md:713-722 App. E.1), with the semantics NCCL/RCCL define (§4 Key Approach:
 *   HetCCL "invokes pure NCCL and RCCL for vendor-local collectives, while handling cross-vendor
 *   coordination in a separate layer"), plus Reduce and All-to-All (App. E.1, NEXT-2).
 *   The hierarchical composition the paper leaves unspecified is read as: reduce within each
 *   device domain, then combine the domain partials across domains (
 *   DESIGN.md reading R1). Per element i the fixed floating-point order is (reading R3):
 *     1. K_k = ranks r with map[r] == k, ascending, k = 0..D-1 (ids dense, reading R4).
 *     2. a_k = widen(x_{K_k[0]}[i]); for each later r in K_k: a_k = a_k (+) widen(x_r[i])
 *        (fold seeded with the first operand, reading R5).
 *     3. P_k = narrow(a_k) if D > 1 else a_k  (16-bit types rounded once per stage, reading R6).
 *     4. y = widen(P_0); for k = 1..D-1: y = y (+) widen(P_k);  Y[i] = narrow(y).
 *   Accumulators: int32 -> uint32 (wraps mod 2^32, reading R8); f32/bf16/f16 -> binary32.
 *   (+): sum = IEEE binary32 round-to-nearest-even add / uint32 add; min/max = fminf/fmaxf
 *   or signed compare (reading R11).
 *
 * Build: gcc -O2 -std=c11 -fno-fast-math -ffp-contract=off -fPIC -shared (x86-64 SSE, FLT_EVAL_METHOD 0).
 */
#include "hetccl_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXR ORACLE_MAX_RANKS

/* ---- element conversions (readings R6, R9, R10) ---- */

static float bf16_to_f32(uint16_t h) { /* exact: bf16 is the top half of a binary32 */
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint16_t f32_to_bf16(float f) { /* round to nearest, ties to even; NaN -> quiet NaN */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu) != 0) return (uint16_t)((u >> 16) | 0x0040u);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

static float f16_to_f32(uint16_t h) { /* exact */
  _Float16 v;
  memcpy(&v, &h, 2);
  return (float)v;
}

static uint16_t f32_to_f16(float f) { /* IEEE conversion: RNE, overflow -> inf, subnormals kept */
  _Float16 v = (_Float16)f;
  uint16_t h;
  memcpy(&h, &v, 2);
  return h;
}

/* ---- the combine operator (+) on accumulators ---- */

static float fop(int op, float a, float b) {
  if (op == ORACLE_SUM) return a + b;
  if (op == ORACLE_MAX) return fmaxf(a, b);
  return fminf(a, b);
}

static uint32_t iop(int op, uint32_t a, uint32_t b) {
  if (op == ORACLE_SUM) return a + b; /* mod 2^32 */
  int32_t sa = (int32_t)a, sb = (int32_t)b;
  if (op == ORACLE_MAX) return (uint32_t)(sa > sb ? sa : sb);
  return (uint32_t)(sa < sb ? sa : sb);
}

static float widen(int dt, const void* p, size_t i) {
  if (dt == ORACLE_F32) return ((const float*)p)[i];
  if (dt == ORACLE_BF16) return bf16_to_f32(((const uint16_t*)p)[i]);
  return f16_to_f32(((const uint16_t*)p)[i]);
}

/* narrow then widen again: the value a 16-bit partial holds once stored in the dtype */
static float round_to_dtype(int dt, float a) {
  if (dt == ORACLE_BF16) return bf16_to_f32(f32_to_bf16(a));
  if (dt == ORACLE_F16) return f16_to_f32(f32_to_f16(a));
  return a;
}

static void store(int dt, void* p, size_t i, float y) {
  if (dt == ORACLE_F32) ((float*)p)[i] = y;
  else if (dt == ORACLE_BF16) ((uint16_t*)p)[i] = f32_to_bf16(y);
  else ((uint16_t*)p)[i] = f32_to_f16(y);
}

/* ---- domain map: K_k lists (reading R4: ids must be dense 0..D-1) ---- */

typedef struct {
  int D;
  int size[MAXR];
  int member[MAXR][MAXR]; /* member[k][j] = j-th rank (ascending) of domain k */
} domains_t;

static int build_domains(int n, const int* map, domains_t* dm) {
  if (n < 1 || n > MAXR || !map) return -1;
  memset(dm, 0, sizeof(*dm));
  int D = 0;
  for (int r = 0; r < n; r++) {
    if (map[r] < 0 || map[r] >= n) return -1;
    if (map[r] + 1 > D) D = map[r] + 1;
  }
  for (int r = 0; r < n; r++) dm->member[map[r]][dm->size[map[r]]++] = r; /* ascending r */
  for (int k = 0; k < D; k++)
    if (dm->size[k] == 0) return -1; /* not dense */
  dm->D = D;
  return 0;
}

static int valid_dtype(int dt) { return dt == ORACLE_INT32 || dt == ORACLE_F32 || dt == ORACLE_BF16 || dt == ORACLE_F16; }
static int valid_op(int op) { return op == ORACLE_SUM || op == ORACLE_MAX || op == ORACLE_MIN; }
static size_t dsize(int dt) { return dt == ORACLE_INT32 || dt == ORACLE_F32 ? 4 : 2; }

/* Y[i] for i in [lo, hi) of the element-wise hierarchical reduction; x[r] indexed from 0 */
static void reduce_range(const domains_t* dm, const void* const* x, void* y, size_t y_off, size_t lo, size_t hi,
                         int dt, int op) {
  int D = dm->D;
  for (size_t i = lo; i < hi; i++) {
    if (dt == ORACLE_INT32) {
      uint32_t P[MAXR];
      for (int k = 0; k < D; k++) {
        uint32_t a = (uint32_t)((const int32_t*)x[dm->member[k][0]])[i];
        for (int j = 1; j < dm->size[k]; j++) a = iop(op, a, (uint32_t)((const int32_t*)x[dm->member[k][j]])[i]);
        P[k] = a; /* narrow is the identity for int32 */
      }
      uint32_t acc = P[0];
      for (int k = 1; k < D; k++) acc = iop(op, acc, P[k]);
      ((int32_t*)y)[y_off + (i - lo)] = (int32_t)acc;
    } else {
      float P[MAXR];
      for (int k = 0; k < D; k++) {
        float a = widen(dt, x[dm->member[k][0]], i);
        for (int j = 1; j < dm->size[k]; j++) a = fop(op, a, widen(dt, x[dm->member[k][j]], i));
        P[k] = (D > 1) ? round_to_dtype(dt, a) : a;
      }
      float acc = P[0];
      for (int k = 1; k < D; k++) acc = fop(op, acc, P[k]);
      store(dt, y, y_off + (i - lo), acc);
    }
  }
}

/* ---- public entry points ---- */

int oracle_allreduce(int nranks, const int* map, const void* const* x, void* y, size_t count, int dtype, int op) {
  domains_t dm;
  if (build_domains(nranks, map, &dm) || !valid_dtype(dtype) || !valid_op(op)) return -1;
  if (count == 0) return 0;
  if (!x || !y) return -1;
  reduce_range(&dm, x, y, 0, 0, count, dtype, op);
  return 0;
}

int oracle_reduce_scatter(int nranks, const int* map, const void* const* x, void* const* y, size_t recvcount,
                          int dtype, int op) {
  domains_t dm;
  if (build_domains(nranks, map, &dm) || !valid_dtype(dtype) || !valid_op(op)) return -1;
  if (recvcount == 0) return 0;
  for (int r = 0; r < nranks; r++) /* rank r receives block r of the reduction */
    reduce_range(&dm, x, y[r], 0, (size_t)r * recvcount, (size_t)(r + 1) * recvcount, dtype, op);
  return 0;
}

int oracle_all_gather(int nranks, const void* const* x, void* const* y, size_t sendcount, int dtype) {
  if (nranks < 1 || nranks > MAXR || !valid_dtype(dtype)) return -1;
  size_t es = dsize(dtype);
  for (int r = 0; r < nranks; r++)
    for (int j = 0; j < nranks; j++) /* out_r[j*R + t] = x_j[t] */
      memcpy((char*)y[r] + (size_t)j * sendcount * es, x[j], sendcount * es);
  return 0;
}

int oracle_broadcast(int nranks, int root, const void* const* x, void* const* y, size_t count, int dtype) {
  if (nranks < 1 || nranks > MAXR || !valid_dtype(dtype) || root < 0 || root >= nranks) return -1;
  size_t es = dsize(dtype);
  for (int r = 0; r < nranks; r++) memcpy(y[r], x[root], count * es); /* out_r = x_root */
  return 0;
}

int oracle_reduce(int nranks, const int* map, int root, const void* const* x, void* y, size_t count, int dtype,
                  int op) {
  if (root < 0 || root >= nranks) return -1;
  return oracle_allreduce(nranks, map, x, y, count, dtype, op); /* out_root = Y */
}

int oracle_all_to_all(int nranks, const void* const* x, void* const* y, size_t blockcount, int dtype) {
  if (nranks < 1 || nranks > MAXR || !valid_dtype(dtype)) return -1;
  size_t es = dsize(dtype), b = blockcount * es;
  for (int i = 0; i < nranks; i++)
    for (int j = 0; j < nranks; j++) /* rank i receives block i of rank j at position j */
      memcpy((char*)y[i] + (size_t)j * b, (const char*)x[j] + (size_t)i * b, b);
  return 0;
}

uint16_t oracle_f32_to_bf16(float f) { return f32_to_bf16(f); }
uint16_t oracle_f32_to_f16(float f) { return f32_to_f16(f); }
float oracle_bf16_to_f32(uint16_t h) { return bf16_to_f32(h); }
float oracle_f16_to_f32(uint16_t h) { return f16_to_f32(h); }
