/* p2_oracle.c — CPU restatement of the reference hot path (TEST INFRASTRUCTURE;
 * see p2_oracle.h).  Deliberately literal: full-region copies, the reference's
 * loop nests and a full-region compare — none of the GPU evaluator's shortcuts
 * (dirty lists, last-writer algebra, staging) — so that it checks them.
 * Built with -ffp-contract=off: acc += av * bv is never fused. */
#include "p2_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

enum { SZ_M, SZ_N, SZ_K, SZ_LDA, SZ_LDB, SZ_LDC, SZ_CN, SZ_CC, SZ_CH, SZ_CW, SZ_CK, SZ_CR, SZ_CS, SZ_COH, SZ_COW };

/* role_value (equivalence.cpp:33-38) */
static int64_t role_value(const oracle_spec* s, const int64_t* sizes, int role, int64_t fallback) {
  int q = s->role_size[role];
  return q < 0 ? fallback : sizes[q];
}

static int array_of_role(const oracle_spec* s, int role) {
  for (int a = 0; a < s->n_arrays; ++a)
    if (s->array_role[a] == role) return a;
  return -1;
}

/* reference_gemm (equivalence.cpp:40-65) */
static int ref_gemm(const oracle_spec* s, const int64_t* sizes, double* const* bufs, const int64_t* lens) {
  const int64_t m = role_value(s, sizes, SZ_M, 0);
  const int64_t n = role_value(s, sizes, SZ_N, 0);
  const int64_t k = role_value(s, sizes, SZ_K, 0);
  const int row = s->layout == 0;
  const int64_t lda = role_value(s, sizes, SZ_LDA, row ? k : m);
  const int64_t ldb = role_value(s, sizes, SZ_LDB, row ? n : k);
  const int64_t ldc = role_value(s, sizes, SZ_LDC, row ? n : m);
  const int ia = array_of_role(s, 0), ib = array_of_role(s, 1), ic = array_of_role(s, 2);
  const double* A = bufs[ia];
  const double* B = bufs[ib];
  double* C = bufs[ic];
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) {
        int64_t ai = row ? i * lda + p : p * lda + i;
        int64_t bi = row ? p * ldb + j : j * ldb + p;
        if (ai < 0 || ai >= lens[ia] || bi < 0 || bi >= lens[ib]) return -1;
        double av = A[ai];
        double bv = B[bi];
        acc += av * bv;
      }
      int64_t ci = row ? i * ldc + j : j * ldc + i;
      if (ci < 0 || ci >= lens[ic]) return -1;
      C[ci] = acc;
    }
  return 0;
}

/* reference_conv2d (equivalence.cpp:67-93) */
static int ref_conv(const oracle_spec* s, const int64_t* sizes, double* const* bufs, const int64_t* lens) {
  const int64_t n = role_value(s, sizes, SZ_CN, 0), c = role_value(s, sizes, SZ_CC, 0);
  const int64_t h = role_value(s, sizes, SZ_CH, 0), w = role_value(s, sizes, SZ_CW, 0);
  const int64_t k = role_value(s, sizes, SZ_CK, 0), r = role_value(s, sizes, SZ_CR, 0);
  const int64_t sw = role_value(s, sizes, SZ_CS, 0);
  const int64_t oh = role_value(s, sizes, SZ_COH, h - r + 1);
  const int64_t ow = role_value(s, sizes, SZ_COW, w - sw + 1);
  const int ii = array_of_role(s, 0), iw = array_of_role(s, 1), io = array_of_role(s, 2);
  const double* in = bufs[ii];
  const double* wt = bufs[iw];
  double* out = bufs[io];
  for (int64_t b = 0; b < n; ++b)
    for (int64_t q = 0; q < k; ++q)
      for (int64_t y = 0; y < oh; ++y)
        for (int64_t x = 0; x < ow; ++x) {
          double acc = 0.0;
          for (int64_t z = 0; z < c; ++z)
            for (int64_t u = 0; u < r; ++u)
              for (int64_t v = 0; v < sw; ++v) {
                int64_t xi = ((b * c + z) * h + y + u) * w + x + v;
                int64_t wi = ((q * c + z) * r + u) * sw + v;
                if (xi < 0 || xi >= lens[ii] || wi < 0 || wi >= lens[iw]) return -1;
                acc += in[xi] * wt[wi];
              }
          int64_t oi = ((b * k + q) * oh + y) * ow + x;
          if (oi < 0 || oi >= lens[io]) return -1;
          out[oi] = acc;
        }
  return 0;
}

int oracle_run_reference(const oracle_spec* s, const int64_t* sizes, double* const* bufs, const int64_t* lens) {
  if (s->semantics == 0) return ref_gemm(s, sizes, bufs, lens);
  if (s->semantics == 1) return ref_conv(s, sizes, bufs, lens);
  return -1;
}

void oracle_verify_binding(const oracle_spec* s, int T, int nI, int nP, const int64_t* ints,
                           const int32_t* is_f32, const int64_t* region_len, const double* const* init,
                           const double* const* fin, const int32_t* test_ok, const uint8_t* arr_map,
                           const uint8_t* size_map, int8_t* fail_t, int8_t* reason) {
  (void)nP;
  double* bufs[4] = {0, 0, 0, 0};
  int64_t lens[4] = {0, 0, 0, 0};
  int64_t sizes[12];
  *fail_t = -1;
  *reason = 0;
  for (int t = 0; t < T; ++t) {
    if (!test_ok[t]) { /* draw failure / original run not Normal (rewriter.cpp:241-251) */
      *fail_t = (int8_t)t;
      *reason = 3;
      goto done;
    }
    for (int q = 0; q < s->n_sizes; ++q) sizes[q] = ints[(int64_t)t * nI + size_map[q]];
    /* run_dispatch checks (rewriter.cpp:136-148) */
    for (int a = 0; a < s->n_arrays; ++a) {
      int64_t extent = 1;
      for (int d = 0; d < s->array_ndims[a]; ++d) {
        int64_t v = sizes[s->array_dims[a][d]];
        if (v < 1) {
          *fail_t = (int8_t)t;
          *reason = 2;
          goto done;
        }
        extent *= v;
      }
      if (region_len[arr_map[a]] < extent) {
        *fail_t = (int8_t)t;
        *reason = 2;
        goto done;
      }
    }
    /* buffers are full-region copies (rewriter.cpp:121) */
    for (int a = 0; a < s->n_arrays; ++a) {
      int p = arr_map[a];
      lens[a] = region_len[p];
      bufs[a] = (double*)realloc(bufs[a], (size_t)lens[a] * sizeof(double));
      memcpy(bufs[a], init[(int64_t)t * nP + p], (size_t)lens[a] * sizeof(double));
    }
    if (oracle_run_reference(s, sizes, bufs, lens) != 0) {
      *fail_t = (int8_t)t;
      *reason = 4;
      goto done;
    }
    /* write-back (rewriter.cpp:152-161) and compare (:264-279) */
    for (int a = 0; a < s->n_arrays; ++a) {
      if (s->array_livein[a]) continue;
      int p = arr_map[a];
      const int f32 = is_f32[p] != 0;
      const double rel = f32 ? 1e-4 : 1e-9, abs_ = f32 ? 1e-6 : 1e-12;
      const double* want = fin[(int64_t)t * nP + p];
      for (int64_t i = 0; i < lens[a]; ++i) {
        double have = f32 ? (double)(float)bufs[a][i] : bufs[a][i];
        if (fabs(have - want[i]) > abs_ + rel * fabs(want[i])) {
          *fail_t = (int8_t)t;
          *reason = 1;
          goto done;
        }
      }
    }
  }
done:
  for (int a = 0; a < 4; ++a) free(bufs[a]);
}

typedef struct {
  const oracle_spec* s;
  int T, nI, nP;
  const int64_t* ints;
  const int32_t* is_f32;
  const int64_t* region_len;
  const double* const* init;
  const double* const* fin;
  const int32_t* test_ok;
  const uint8_t* arr_map;
  const uint8_t* size_map;
  int64_t n;
  int8_t* fail_t;
  int8_t* reason;
  atomic_llong next;
} many_args;

static void* many_worker(void* p) {
  many_args* a = (many_args*)p;
  for (;;) {
    long long b = atomic_fetch_add(&a->next, 1);
    if (b >= a->n) break;
    oracle_verify_binding(a->s, a->T, a->nI, a->nP, a->ints, a->is_f32, a->region_len, a->init, a->fin,
                          a->test_ok, a->arr_map + b * a->s->n_arrays, a->size_map + b * a->s->n_sizes,
                          a->fail_t + b, a->reason + b);
  }
  return NULL;
}

void oracle_verify_many(const oracle_spec* s, int T, int nI, int nP, const int64_t* ints, const int32_t* is_f32,
                        const int64_t* region_len, const double* const* init, const double* const* fin,
                        const int32_t* test_ok, const uint8_t* arr_map, const uint8_t* size_map, int64_t n,
                        int threads, int8_t* fail_t, int8_t* reason) {
  many_args a = {s, T, nI, nP, ints, is_f32, region_len, init, fin, test_ok, arr_map, size_map, n, fail_t, reason, 0};
  if (threads < 1) threads = 1;
  pthread_t th[256];
  if (threads > 256) threads = 256;
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, many_worker, &a);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
}

/* profitability::cpu_gemm (profitability.cpp:14-21) */
void oracle_cpu_gemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      float acc = 0.0f;
      for (int64_t p = 0; p < k; ++p) acc += a[i * k + p] * b[p * n + j];
      c[i * n + j] = acc;
    }
}

/* profitability::xpu_stripe / xpu_gemm (profitability.cpp:25-63) */
enum { kTile = 64 };
typedef struct {
  const float *a, *b;
  float* c;
  int64_t m, n, k, lo, hi;
} stripe_args;

static void* xpu_stripe(void* p) {
  stripe_args* s = (stripe_args*)p;
  const float *a = s->a, *b = s->b;
  float* c = s->c;
  const int64_t n = s->n, k = s->k;
  for (int64_t i = s->lo; i < s->hi; ++i)
    for (int64_t j = 0; j < n; ++j) c[i * n + j] = 0.0f;
  for (int64_t i0 = s->lo; i0 < s->hi; i0 += kTile)
    for (int64_t p0 = 0; p0 < k; p0 += kTile)
      for (int64_t j0 = 0; j0 < n; j0 += kTile) {
        const int64_t im = i0 + kTile < s->hi ? i0 + kTile : s->hi;
        const int64_t pm = p0 + kTile < k ? p0 + kTile : k;
        const int64_t jm = j0 + kTile < n ? j0 + kTile : n;
        for (int64_t i = i0; i < im; ++i)
          for (int64_t p = p0; p < pm; ++p) {
            const float av = a[i * k + p];
            for (int64_t j = j0; j < jm; ++j) c[i * n + j] += av * b[p * n + j];
          }
      }
  return NULL;
}

void oracle_xpu_gemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int threads) {
  int64_t nthreads = threads < 1 ? 1 : threads;
  int64_t tiles = (m + kTile - 1) / kTile;
  if (nthreads > tiles) nthreads = tiles;
  if (nthreads <= 1) {
    stripe_args s = {a, b, c, m, n, k, 0, m};
    xpu_stripe(&s);
    return;
  }
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  stripe_args args[256];
  const int64_t chunk = (m + nthreads - 1) / nthreads;
  int started = 0;
  for (int64_t t = 0; t < nthreads; ++t) {
    int64_t lo = t * chunk, hi = lo + chunk < m ? lo + chunk : m;
    if (lo >= hi) break;
    args[t] = (stripe_args){a, b, c, m, n, k, lo, hi};
    pthread_create(&th[t], NULL, xpu_stripe, &args[t]);
    ++started;
  }
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

uint64_t oracle_fnv1a(const void* p, int64_t nbytes) {
  const unsigned char* b = (const unsigned char*)p;
  uint64_t h = 1469598103934665603ULL;
  for (int64_t i = 0; i < nbytes; ++i) {
    h ^= b[i];
    h *= 1099511628211ULL;
  }
  return h;
}
