/*
 * pool.c — persistent pthread pool for the CPU oracle (TEST INFRASTRUCTURE:
 * only tests/, __graft_entry__.smoke() and bench.py's CPU legs load the
 * oracle library).  Workers sleep on a condition variable between loops; a
 * loop hands each thread one contiguous span [n*t/nt, n*(t+1)/nt) and the
 * caller runs span 0 itself.  Spawning threads per call cost ~100 us, which
 * the CPU SD loop (thousands of small projections per iteration) cannot
 * afford.
 */
#include "pool.h"

#include <pthread.h>
#include <stdlib.h>

#define MAX_THREADS 256

static int g_threads = 1;

static struct {
  pthread_mutex_t mu;
  pthread_cond_t go, done;
  pthread_t th[MAX_THREADS];
  int started;      /* workers alive */
  uint64_t gen;     /* loop generation */
  int pending;      /* workers still running the current loop */
  oracle_row_fn fn;
  void* ctx;
  int64_t n;
  int nt;           /* threads in the current loop */
} P = {.mu = PTHREAD_MUTEX_INITIALIZER, .go = PTHREAD_COND_INITIALIZER, .done = PTHREAD_COND_INITIALIZER};

static void run_span(int t) {
  const int64_t lo = P.n * t / P.nt, hi = P.n * (t + 1) / P.nt;
  for (int64_t i = lo; i < hi; ++i) P.fn(P.ctx, i);
}

static void* worker(void* arg) {
  const int t = (int)(intptr_t)arg;
  uint64_t seen = 0;
  pthread_mutex_lock(&P.mu);
  for (;;) {
    while (P.gen == seen) pthread_cond_wait(&P.go, &P.mu);
    seen = P.gen;
    const int active = t < P.nt;
    pthread_mutex_unlock(&P.mu);
    if (active) run_span(t);
    pthread_mutex_lock(&P.mu);
    if (active && --P.pending == 0) pthread_cond_signal(&P.done);
  }
  return NULL;
}

void oracle_set_threads(int n) {
  g_threads = n < 1 ? 1 : (n > MAX_THREADS ? MAX_THREADS : n);
}

int oracle_num_threads(void) { return g_threads; }

void oracle_parallel_for(int64_t n, oracle_row_fn fn, void* ctx) {
  int nt = g_threads;
  if (nt > n) nt = (int)(n > 0 ? n : 1);
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) fn(ctx, i);
    return;
  }
  pthread_mutex_lock(&P.mu);
  while (P.started < nt - 1) {
    /* worker k runs span k + 1 (the caller runs span 0) */
    pthread_create(&P.th[P.started], NULL, worker, (void*)(intptr_t)(P.started + 1));
    ++P.started;
  }
  P.fn = fn;
  P.ctx = ctx;
  P.n = n;
  P.nt = nt;
  P.pending = nt - 1;
  ++P.gen;
  pthread_cond_broadcast(&P.go);
  pthread_mutex_unlock(&P.mu);
  run_span(0);
  pthread_mutex_lock(&P.mu);
  while (P.pending > 0) pthread_cond_wait(&P.done, &P.mu);
  pthread_mutex_unlock(&P.mu);
}
