/*
 * chw_oracle.c — plain-C restatement of the reference CHW algorithm.
 *
 * TEST INFRASTRUCTURE ONLY (see chw_oracle.h).  Each function follows the
 * reference loop structure literally, citing the lines it restates, so that
 * floating-point results are bitwise identical to the reference's
 * (checked against oracle/_ref and tests/golden/ in tests/test_oracle.py).
 *
 * Build: oracle/Makefile (gcc -std=c11 -O3 -DNDEBUG -fPIC -shared).
 * No FMA contraction is possible: x86-64 baseline ISA, -ffp-contract=off.
 */
#include "chw_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* common.hpp:29 */
static const double kInvSqrt2 = 0.70710678118654752440;

/* common.hpp:22-25 */
static int is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }
static int level_of(size_t n) {
  int m = 0;
  while (((size_t)1 << (m + 1)) <= n && (m + 1) < (int)(8 * sizeof(size_t))) ++m;
  return m;
}

uint64_t chw_oracle_bit_reverse(uint64_t v, int bits) {
  /* orderings.hpp:45-52 */
  uint64_t r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (v & 1u);
    v >>= 1;
  }
  return r;
}

/* The reference templates (transforms.hpp) are instantiated for int64 and
 * double (common.hpp:19-20); the macro below emits both from one text.
 * IS_FP selects the `if constexpr (is_floating_point_v<T>)` branches. */
#define CHW_ORACLE_DEFINE(T, SFX, IS_FP)                                                        \
  /* transforms.hpp:49-80 — haar_forward_inplace. */                                        \
  static void haar_core_##SFX(T* x, size_t n, int ortho, T* scratch, uint64_t* adds,          \
                              uint64_t* mults) {                                              \
    for (size_t len = n; len >= 2; len >>= 1) {                                               \
      const size_t half = len / 2;                                                            \
      for (size_t i = 0; i < half; ++i) {                                                     \
        T s = x[2 * i] + x[2 * i + 1];                                                        \
        T d = x[2 * i] - x[2 * i + 1];                                                        \
        if (IS_FP && ortho) {                                                                 \
          s = (T)(s * kInvSqrt2);                                                             \
          d = (T)(d * kInvSqrt2);                                                             \
        }                                                                                     \
        x[i] = s; /* write index trails the read pair */                                      \
        scratch[i] = d;                                                                       \
      }                                                                                       \
      memcpy(x + half, scratch, half * sizeof(T));                                            \
      if (adds) *adds += len;                                                                 \
      if (mults && ortho) *mults += len;                                                      \
    }                                                                                         \
  }                                                                                           \
  static int check_##SFX(size_t n, int mode) {                                                \
    if (!is_pow2(n)) return -1;               /* common.hpp:31-36 */                          \
    if (!(IS_FP) && mode == 0) return -2;     /* common.hpp:38-46 */                          \
    return 0;                                                                                 \
  }                                                                                           \
  int chw_oracle_haar_forward_##SFX(T* x, size_t n, int mode, uint64_t* adds,                 \
                                    uint64_t* mults) {                                        \
    int rc = check_##SFX(n, mode);                                                            \
    if (rc) return rc;                                                                        \
    T* scratch = (T*)malloc((n / 2 + 1) * sizeof(T));                                         \
    haar_core_##SFX(x, n, mode == 0, scratch, adds, mults);                                   \
    free(scratch);                                                                            \
    return 0;                                                                                 \
  }                                                                                           \
  /* transforms.hpp:126-143 — chw_forward_inplace: one full Haar transform, then for r =    \
   * 1..m-1 a Haar transform on every stage_blocks(m, r) slice (transforms.hpp:30-42:       \
   * offset q*2*size + size, size 2^(m-r), q < 2^(r-1)), in stage order. */                   \
  int chw_oracle_chw_forward_##SFX(T* x, size_t n, int mode, uint64_t* adds,                  \
                                   uint64_t* mults) {                                         \
    int rc = check_##SFX(n, mode);                                                            \
    if (rc) return rc;                                                                        \
    const int m = level_of(n);                                                                \
    T* scratch = (T*)malloc((n / 2 + 1) * sizeof(T));                                         \
    haar_core_##SFX(x, n, mode == 0, scratch, adds, mults);                                   \
    for (int r = 1; r <= m - 1; ++r) {                                                        \
      const size_t size = (size_t)1 << (m - r);                                               \
      for (size_t q = 0; q < ((size_t)1 << (r - 1)); ++q) {                                   \
        haar_core_##SFX(x + q * 2 * size + size, size, mode == 0, scratch, adds, mults);      \
      }                                                                                       \
    }                                                                                         \
    free(scratch);                                                                            \
    return 0;                                                                                 \
  }                                                                                           \
  /* transforms.hpp:147-172 — fwht_natural_inplace. */                                        \
  int chw_oracle_fwht_natural_##SFX(T* x, size_t n, int mode) {                               \
    int rc = check_##SFX(n, mode);                                                            \
    if (rc) return rc;                                                                        \
    for (size_t h = 1; h < n; h <<= 1) {                                                      \
      for (size_t i = 0; i < n; i += 2 * h) {                                                 \
        for (size_t j = i; j < i + h; ++j) {                                                  \
          T s = x[j] + x[j + h];                                                              \
          T d = x[j] - x[j + h];                                                              \
          if (IS_FP && mode == 0) {                                                           \
            s = (T)(s * kInvSqrt2);                                                           \
            d = (T)(d * kInvSqrt2);                                                           \
          }                                                                                   \
          x[j] = s;                                                                           \
          x[j + h] = d;                                                                       \
        }                                                                                     \
      }                                                                                       \
    }                                                                                         \
    return 0;                                                                                 \
  }                                                                                           \
  /* transforms.hpp:177-185 — natural WHT then in-place bit-reversal swaps. */                \
  int chw_oracle_fwht_dyadic_##SFX(T* x, size_t n, int mode) {                                \
    int rc = chw_oracle_fwht_natural_##SFX(x, n, mode);                                       \
    if (rc) return rc;                                                                        \
    const int m = level_of(n);                                                                \
    for (size_t i = 0; i < n; ++i) {                                                          \
      const size_t j = (size_t)chw_oracle_bit_reverse(i, m);                                  \
      if (i < j) {                                                                            \
        T t = x[i];                                                                           \
        x[i] = x[j];                                                                          \
        x[j] = t;                                                                             \
      }                                                                                       \
    }                                                                                         \
    return 0;                                                                                 \
  }                                                                                           \
  /* transforms.hpp:190-198 — dyadic WHT on each scale block [2^j, 2^(j+1)), j = 1..m-1. */   \
  int chw_oracle_haar_walsh_forward_##SFX(T* x, size_t n, int mode) {                         \
    int rc = check_##SFX(n, mode);                                                            \
    if (rc) return rc;                                                                        \
    const int m = level_of(n);                                                                \
    for (int j = 1; j <= m - 1; ++j) {                                                        \
      chw_oracle_fwht_dyadic_##SFX(x + ((size_t)1 << j), (size_t)1 << j, mode);               \
    }                                                                                         \
    return 0;                                                                                 \
  }

CHW_ORACLE_DEFINE(double, f64, 1)
CHW_ORACLE_DEFINE(int64_t, i64, 0)

/* transforms.hpp:85-120 — haar_inverse_inplace (float branch). */
int chw_oracle_haar_inverse_f64(double* x, size_t n, int mode) {
  if (!is_pow2(n)) return -1;
  double* scratch = (double*)malloc((n / 2 + 1) * sizeof(double));
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len / 2;
    memcpy(scratch, x, half * sizeof(double));
    for (size_t i = 0; i < half; ++i) {
      const double s = scratch[i];
      const double d = x[half + i];
      if (mode == 0) {
        x[2 * i] = (s + d) * kInvSqrt2;
        x[2 * i + 1] = (s - d) * kInvSqrt2;
      } else {
        x[2 * i] = (s + d) / 2;
        x[2 * i + 1] = (s - d) / 2;
      }
    }
  }
  free(scratch);
  return 0;
}

/* transforms.hpp:85-120 — integer branch with the parity check (StructureError). */
int chw_oracle_haar_inverse_i64(int64_t* x, size_t n, int mode) {
  if (!is_pow2(n)) return -1;
  if (mode == 0) return -2;
  int64_t* scratch = (int64_t*)malloc((n / 2 + 1) * sizeof(int64_t));
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len / 2;
    memcpy(scratch, x, half * sizeof(int64_t));
    for (size_t i = 0; i < half; ++i) {
      const int64_t s = scratch[i];
      const int64_t d = x[half + i];
      const int64_t sum = s + d;
      if (sum & 1) {
        free(scratch);
        return -3;
      }
      x[2 * i] = sum / 2;
      x[2 * i + 1] = (s - d) / 2;
    }
  }
  free(scratch);
  return 0;
}

/* transforms.hpp:202-210 — normalize_inplace: x *= 1/sqrt(2^m). */
int chw_oracle_normalize_f64(double* x, size_t n, int m) {
  if (m < 0 || m > 62 || n != ((size_t)1 << m)) return -1;
  double p = 1.0;
  for (int i = 0; i < m; ++i) p *= 2.0; /* ldexp(1.0, m), exact */
  /* 1.0 / sqrt(p): sqrt is correctly rounded (IEEE), as in the reference. */
  const double c = 1.0 / sqrt(p);
  for (size_t i = 0; i < n; ++i) x[i] *= c;
  return 0;
}

/* level-synchronous butterfly network + bit reversal. */
int chw_oracle_network_f64(double* x, size_t n, int mode) {
  if (!is_pow2(n)) return -1;
  const int m = level_of(n);
  for (int t = 0; t < m; ++t) {
    const size_t h = (size_t)1 << t;
    for (size_t j = 0; j < n; ++j) {
      if (j & h) continue;
      const double a = x[j], b = x[j | h];
      double s = a + b, d = a - b;
      if (mode == 0) {
        s *= kInvSqrt2;
        d *= kInvSqrt2;
      }
      x[j] = s;
      x[j | h] = d;
    }
  }
  for (size_t i = 0; i < n; ++i) {
    const size_t j = (size_t)chw_oracle_bit_reverse(i, m);
    if (i < j) {
      double t = x[i];
      x[i] = x[j];
      x[j] = t;
    }
  }
  return 0;
}

int chw_oracle_online_cores(void) {
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}

/* Batched drivers: rows statically partitioned across threads, each with its
 * own scratch (SPEC.md:233 — disjoint buffers are safe to transform
 * concurrently). */
typedef struct {
  void* base;
  size_t row0, row1, n;
  int mode, is_fp;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (size_t r = j->row0; r < j->row1; ++r) {
    if (j->is_fp)
      chw_oracle_chw_forward_f64((double*)j->base + r * j->n, j->n, j->mode, NULL, NULL);
    else
      chw_oracle_chw_forward_i64((int64_t*)j->base + r * j->n, j->n, j->mode, NULL, NULL);
  }
  return NULL;
}

static int run_batch(void* x, size_t rows, size_t n, int mode, int threads, int is_fp) {
  if (!is_pow2(n)) return -1;
  if (!is_fp && mode == 0) return -2;
  if (threads <= 0) threads = chw_oracle_online_cores();
  if ((size_t)threads > rows) threads = rows ? (int)rows : 1;
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  batch_job* jobs = (batch_job*)calloc((size_t)threads, sizeof(batch_job));
  for (int t = 0; t < threads; ++t) {
    jobs[t].base = x;
    jobs[t].row0 = rows * (size_t)t / (size_t)threads;
    jobs[t].row1 = rows * (size_t)(t + 1) / (size_t)threads;
    jobs[t].n = n;
    jobs[t].mode = mode;
    jobs[t].is_fp = is_fp;
    pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

int chw_oracle_chw_batch_f64(double* x, size_t rows, size_t n, int mode, int threads) {
  return run_batch(x, rows, n, mode, threads, 1);
}
int chw_oracle_chw_batch_i64(int64_t* x, size_t rows, size_t n, int mode, int threads) {
  return run_batch(x, rows, n, mode, threads, 0);
}
