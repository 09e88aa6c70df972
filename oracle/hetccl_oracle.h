/*
 * hetccl_oracle.h — CPU oracle for the hierarchical collectives. TEST INFRASTRUCTURE ONLY
 * (see hetccl_oracle.c for what it computes and the passages it follows). No CUDA, no code shared
 * with the product path. All buffers are host memory; x[r] is rank r's input, y / y[r] outputs.
 * Return 0 on success, -1 on an invalid argument (bad map, dtype, op, root, or rank count).
 */
#ifndef HETCCL_ORACLE_H
#define HETCCL_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_MAX_RANKS 64

/* dtype codes (numerically NCCL's, written out independently here) */
enum { ORACLE_INT32 = 2, ORACLE_F16 = 6, ORACLE_F32 = 7, ORACLE_BF16 = 9 };
/* reduction operators */
enum { ORACLE_SUM = 0, ORACLE_MAX = 2, ORACLE_MIN = 3 };

/* Y = hierarchical reduction of x[0..nranks) (one output array, identical on every rank) */
int oracle_allreduce(int nranks, const int* map, const void* const* x, void* y, size_t count, int dtype, int op);
/* y[r] = Y[r*recvcount .. (r+1)*recvcount) ; x[r] holds nranks*recvcount elements */
int oracle_reduce_scatter(int nranks, const int* map, const void* const* x, void* const* y, size_t recvcount,
                          int dtype, int op);
/* y[r][j*sendcount + t] = x[j][t] */
int oracle_all_gather(int nranks, const void* const* x, void* const* y, size_t sendcount, int dtype);
/* y[r] = x[root] */
int oracle_broadcast(int nranks, int root, const void* const* x, void* const* y, size_t count, int dtype);
/* y (root's output) = Y */
int oracle_reduce(int nranks, const int* map, int root, const void* const* x, void* y, size_t count, int dtype,
                  int op);
/* y[i][j*b + t] = x[j][i*b + t] */
int oracle_all_to_all(int nranks, const void* const* x, void* const* y, size_t blockcount, int dtype);

uint16_t oracle_f32_to_bf16(float f);
uint16_t oracle_f32_to_f16(float f);
float oracle_bf16_to_f32(uint16_t h);
float oracle_f16_to_f32(uint16_t h);

#ifdef __cplusplus
}
#endif
#endif
