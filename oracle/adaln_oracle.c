/*
 * adaln_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's f64 AdaLN
 * kernels, used by tests/ as the parity checker and by bench.py as the CPU baseline (the
 * reference arm).  Never linked into or called by the product path.
 *
 * Restates /root/reference/pkg/src/adaptiveload/adaln/_kernels_numba.py operation by operation
 * (same association order, IEEE double, no contraction -> bit-identical to the numba backend,
 * pinned against the reference's own outputs in tests/golden/):
 *   oracle_forward        <- _forward_kernel        _kernels_numba.py:18-34
 *   oracle_backward_dx    <- _backward_dx_kernel    _kernels_numba.py:45-62
 *   oracle_reduce_naive   <- _reduce_naive_kernel   _kernels_numba.py:71-83
 *   oracle_dtile_reduce   <- _dtile_kernel_f64/f32  _kernels_numba.py:94-127
 *   oracle_as_f64_*       <- _as_f64                adaln/__init__.py:81-85 (cast + isfinite)
 *
 * `threads` > 1 parallelises with pthreads without changing any per-element operation order:
 * forward / dx split rows (rows are independent); the reductions split feature columns and
 * every feature still accumulates rows in ascending order (the reference's order).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#define ORACLE_API __attribute__((visibility("default")))

static int nthreads(int t) {
  if (t > 0) return t;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}

ORACLE_API int oracle_max_threads(void) { return nthreads(0); }

/* ---- minimal static parallel-for over [0, n): contiguous chunks, one per thread ---- */
typedef void (*range_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t begin, end;
} task_t;

static void* run_task(void* p) {
  task_t* t = (task_t*)p;
  if (t->begin < t->end) t->fn(t->ctx, t->begin, t->end);
  return NULL;
}

static void parallel_for(int64_t n, int threads, range_fn fn, void* ctx) {
  int nt = nthreads(threads);
  if (nt > 256) nt = 256;
  if (nt > n) nt = (int)(n > 0 ? n : 1);
  if (nt <= 1) {
    if (n > 0) fn(ctx, 0, n);
    return;
  }
  pthread_t tid[256];
  task_t task[256];
  for (int i = 0; i < nt; ++i) {
    task[i].fn = fn;
    task[i].ctx = ctx;
    task[i].begin = n * i / nt;
    task[i].end = n * (i + 1) / nt;
  }
  for (int i = 1; i < nt; ++i) pthread_create(&tid[i], NULL, run_task, &task[i]);
  run_task(&task[0]);
  for (int i = 1; i < nt; ++i) pthread_join(tid[i], NULL);
}

/* _forward_kernel: two-pass population variance, eps inside sqrt, y=(x-m)*r*(1+scale)+shift */
typedef struct {
  const double *x, *scale, *shift;
  double eps;
  int64_t d;
  double *y, *mu, *rstd;
} fwd_ctx;

static void fwd_rows(void* p, int64_t n0, int64_t n1) {
  const fwd_ctx* c = (const fwd_ctx*)p;
  const int64_t d = c->d;
  for (int64_t n = n0; n < n1; ++n) {
    const double* xr = c->x + n * d;
    double s = 0.0;
    for (int64_t j = 0; j < d; ++j) s += xr[j];
    const double m = s / (double)d;
    double v = 0.0;
    for (int64_t j = 0; j < d; ++j) {
      const double t = xr[j] - m;
      v += t * t;
    }
    const double r = 1.0 / sqrt(v / (double)d + c->eps);
    c->mu[n] = m;
    c->rstd[n] = r;
    double* yr = c->y + n * d;
    for (int64_t j = 0; j < d; ++j) yr[j] = (xr[j] - m) * r * (1.0 + c->scale[j]) + c->shift[j];
  }
}

ORACLE_API void oracle_forward(const double* x, const double* scale, const double* shift,
                               double eps, int64_t n_rows, int64_t d, double* y, double* mu,
                               double* rstd, int threads) {
  fwd_ctx c = {x, scale, shift, eps, d, y, mu, rstd};
  parallel_for(n_rows, threads, fwd_rows, &c);
}

/* _backward_dx_kernel */
typedef struct {
  const double *dy, *x, *scale, *mu, *rstd;
  int64_t d;
  double* dx;
} dx_ctx;

static void dx_rows(void* p, int64_t n0, int64_t n1) {
  const dx_ctx* c = (const dx_ctx*)p;
  const int64_t d = c->d;
  for (int64_t n = n0; n < n1; ++n) {
    const double* xr = c->x + n * d;
    const double* gr = c->dy + n * d;
    const double m = c->mu[n], r = c->rstd[n];
    double gs = 0.0, gxs = 0.0;
    for (int64_t j = 0; j < d; ++j) {
      const double g = gr[j] * (1.0 + c->scale[j]);
      gs += g;
      gxs += g * (xr[j] - m) * r;
    }
    const double g_mean = gs / (double)d;
    const double gx_mean = gxs / (double)d;
    double* o = c->dx + n * d;
    for (int64_t j = 0; j < d; ++j) {
      const double g = gr[j] * (1.0 + c->scale[j]);
      const double xh = (xr[j] - m) * r;
      o[j] = r * (g - g_mean - xh * gx_mean);
    }
  }
}

ORACLE_API void oracle_backward_dx(const double* dy, const double* x, const double* scale,
                                   const double* mu, const double* rstd, int64_t n_rows,
                                   int64_t d, double* dx, int threads) {
  dx_ctx c = {dy, x, scale, mu, rstd, d, dx};
  parallel_for(n_rows, threads, dx_rows, &c);
}

/* _reduce_naive_kernel: per feature, rows ascending.  Threads own blocks of whole feature
 * columns; inside a block the row loop is outermost (cache friendly, same per-feature order). */
#define COL_BLOCK 64
typedef struct {
  const double *dy, *x, *mu, *rstd;
  int64_t n_rows, d;
  double *dscale, *dshift;
} red_ctx;

static void naive_blocks(void* p, int64_t b0, int64_t b1) {
  const red_ctx* c = (const red_ctx*)p;
  const int64_t d = c->d;
  for (int64_t b = b0; b < b1; ++b) {
    const int64_t j0 = b * COL_BLOCK;
    const int64_t j1 = j0 + COL_BLOCK < d ? j0 + COL_BLOCK : d;
    for (int64_t j = j0; j < j1; ++j) {
      c->dscale[j] = 0.0;
      c->dshift[j] = 0.0;
    }
    for (int64_t n = 0; n < c->n_rows; ++n) {
      const double m = c->mu[n], r = c->rstd[n];
      const double* xr = c->x + n * d;
      const double* gr = c->dy + n * d;
      for (int64_t j = j0; j < j1; ++j) {
        const double xh = (xr[j] - m) * r;
        c->dshift[j] += gr[j];
        c->dscale[j] += gr[j] * xh;
      }
    }
  }
}

ORACLE_API void oracle_reduce_naive(const double* dy, const double* x, const double* mu,
                                    const double* rstd, int64_t n_rows, int64_t d,
                                    double* dscale, double* dshift, int threads) {
  red_ctx c = {dy, x, mu, rstd, n_rows, d, dscale, dshift};
  parallel_for((d + COL_BLOCK - 1) / COL_BLOCK, threads, naive_blocks, &c);
}

/* _dtile_kernel_f64 / _dtile_kernel_f32: feature-outer, n-tiles ascending. */
typedef struct {
  red_ctx r;
  int64_t d_tile, n_tile;
  int fp32_accum;
} dtile_ctx;

static void dtile_tiles(void* p, int64_t t0, int64_t t1) {
  const dtile_ctx* c = (const dtile_ctx*)p;
  const int64_t d = c->r.d, n_rows = c->r.n_rows, n_tile = c->n_tile;
  const double *x = c->r.x, *dy = c->r.dy, *mu = c->r.mu, *rstd = c->r.rstd;
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t d0 = t * c->d_tile;
    const int64_t d1 = d0 + c->d_tile < d ? d0 + c->d_tile : d;
    for (int64_t j = d0; j < d1; ++j) {
      if (c->fp32_accum) {
        float acc_sh = 0.0f, acc_sc = 0.0f;
        for (int64_t n0 = 0; n0 < n_rows; n0 += n_tile) {
          const int64_t n1 = n0 + n_tile < n_rows ? n0 + n_tile : n_rows;
          for (int64_t n = n0; n < n1; ++n) {
            const double xh = (x[n * d + j] - mu[n]) * rstd[n];
            acc_sh = acc_sh + (float)dy[n * d + j];
            acc_sc = acc_sc + (float)(dy[n * d + j] * xh);
          }
        }
        c->r.dshift[j] = (double)acc_sh;
        c->r.dscale[j] = (double)acc_sc;
      } else {
        double acc_sh = 0.0, acc_sc = 0.0;
        for (int64_t n0 = 0; n0 < n_rows; n0 += n_tile) {
          const int64_t n1 = n0 + n_tile < n_rows ? n0 + n_tile : n_rows;
          for (int64_t n = n0; n < n1; ++n) {
            const double xh = (x[n * d + j] - mu[n]) * rstd[n];
            acc_sh += dy[n * d + j];
            acc_sc += dy[n * d + j] * xh;
          }
        }
        c->r.dshift[j] = acc_sh;
        c->r.dscale[j] = acc_sc;
      }
    }
  }
}

ORACLE_API void oracle_dtile_reduce(const double* dy, const double* x, const double* mu,
                                    const double* rstd, int64_t n_rows, int64_t d,
                                    int64_t d_tile, int64_t n_tile, int fp32_accum,
                                    double* dscale, double* dshift, int threads) {
  dtile_ctx c = {{dy, x, mu, rstd, n_rows, d, dscale, dshift}, d_tile, n_tile, fp32_accum};
  parallel_for((d + d_tile - 1) / d_tile, threads, dtile_tiles, &c);
}

/* _as_f64 for the dtypes the GPU path takes: widen to double and scan for NaN/Inf. */
typedef struct {
  const void* in;
  int kind; /* 0 bf16, 1 f32 */
  double* out;
  int bad;
} cast_ctx;

static void cast_range(void* p, int64_t i0, int64_t i1) {
  cast_ctx* c = (cast_ctx*)p;
  int bad = 0;
  for (int64_t i = i0; i < i1; ++i) {
    double v;
    if (c->kind == 0) {
      uint32_t u = (uint32_t)((const uint16_t*)c->in)[i] << 16;
      float f;
      memcpy(&f, &u, sizeof f);
      v = (double)f;
    } else {
      v = (double)((const float*)c->in)[i];
    }
    c->out[i] = v;
    bad |= !isfinite(v);
  }
  __atomic_fetch_or(&c->bad, bad, __ATOMIC_RELAXED);
}

static int as_f64(const void* in, int kind, int64_t count, double* out, int threads) {
  cast_ctx c;
  memset(&c, 0, sizeof c);
  c.in = in;
  c.kind = kind;
  c.out = out;
  parallel_for(count, threads, cast_range, &c);
  return c.bad;
}

/* Returns 1 if any element is non-finite (the reference raises NonFiniteInput then). */
ORACLE_API int oracle_as_f64_bf16(const uint16_t* in, int64_t count, double* out, int threads) {
  return as_f64(in, 0, count, out, threads);
}

ORACLE_API int oracle_as_f64_f32(const float* in, int64_t count, double* out, int threads) {
  return as_f64(in, 1, count, out, threads);
}
