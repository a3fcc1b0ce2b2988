/*
 * pool.h — persistent worker pool of the CPU oracle (TEST INFRASTRUCTURE;
 * see spmoe_oracle.c).  Every parallel loop splits an index range into
 * contiguous spans, one per thread; each index is computed independently
 * in a fixed order, so results never depend on the thread count.
 */
#ifndef SPMOE_ORACLE_POOL_H
#define SPMOE_ORACLE_POOL_H

#include <stdint.h>

typedef void (*oracle_row_fn)(void* ctx, int64_t i);

void oracle_set_threads(int n);
int oracle_num_threads(void);
void oracle_parallel_for(int64_t n, oracle_row_fn fn, void* ctx);

#endif
