/*
 * oracle/kernels.c -- CPU restatement of the four tuned kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library,
 * and only as the checker or the CPU baseline -- never as the product
 * path.  Parity status: the reference (tunescape, pure Python) contains
 * no kernel arithmetic (SURVEY.md §0.5, §8c "Kernel arithmetic: parity
 * unpinned"); these functions restate the mathematical definitions of
 * SURVEY.md §8(a) row a19 and are pinned by the known-answer tests in
 * tests/test_oracle.py (delta filter = identity, constant field = fixed
 * point, zero shifts = channel sum, identity matrix) and by an
 * independent float64 numpy computation.
 *
 * Every function uses the same fp32 operation order as the CUDA kernels
 * (explicit fmaf / no contraction; build with -ffp-contract=off), so the
 * GPU results are expected to match BIT-FOR-BIT.  a pthread parallel-for
 * splits independent outputs only, which keeps the results deterministic.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

/* ---- a tiny static parallel-for over [0, n) on pthreads (the image has
 * no libgomp).  Deterministic: every output is computed by exactly one
 * thread with the same sequential arithmetic. */
static int g_threads = 0;

void oracle_set_threads(int n) { g_threads = n; }

int oracle_threads(void) {
  if (g_threads > 0) return g_threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

typedef void (*range_fn)(void* ctx, int lo, int hi);
typedef struct {
  range_fn fn;
  void* ctx;
  int lo, hi;
} job_t;

static void* run_job(void* p) {
  job_t* j = (job_t*)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

static void parallel_for(int n, range_fn fn, void* ctx) {
  int t = oracle_threads();
  if (t > n) t = n;
  if (t <= 1) {
    fn(ctx, 0, n);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)t);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)t);
  for (int i = 0; i < t; ++i) {
    jobs[i].fn = fn;
    jobs[i].ctx = ctx;
    jobs[i].lo = (int)((long long)n * i / t);
    jobs[i].hi = (int)((long long)n * (i + 1) / t);
    pthread_create(&th[i], NULL, run_job, &jobs[i]);
  }
  for (int i = 0; i < t; ++i) pthread_join(th[i], NULL);
  free(th);
  free(jobs);
}

/* out[y][x] = sum_{i<fh, j<fw} in[(y+i)*pitch + x+j] * f[i*fw+j], fmaf chain
 * in (i, j) row-major order (kernels/convolution.cu). */
typedef struct {
  float* out;
  const float* in;
  const float* f;
  int pitch, w, fw, fh;
} conv_ctx;

static void conv_rows(void* p, int y0, int y1) {
  conv_ctx* c = (conv_ctx*)p;
  float* out = c->out;
  const float* in = c->in;
  const float* f = c->f;
  const int pitch = c->pitch, w = c->w, fw = c->fw, fh = c->fh;
  for (int y = y0; y < y1; ++y) {
    for (int x = 0; x < w; ++x) {
      float acc = 0.f;
      for (int i = 0; i < fh; ++i) {
        const float* row = in + (size_t)(y + i) * pitch + x;
        for (int j = 0; j < fw; ++j) acc = fmaf(row[j], f[i * fw + j], acc);
      }
      out[(size_t)y * w + x] = acc;
    }
  }
}

void oracle_convolution(float* out, const float* in, int pitch, int w, int h, const float* f,
                        int fw, int fh) {
  conv_ctx c = {out, in, f, pitch, w, fw, fh};
  parallel_for(h, conv_rows, &c);
}

/* One Rodinia hotspot step, clamped boundary, fixed operation order
 * (kernels/hotspot.cu). */
typedef struct {
  float* out;
  const float *tin, *power;
  int w, h;
  float sdc, rx1, ry1, rz1, amb;
} hs_ctx;

static void hotspot_rows(void* p, int y0, int y1) {
  hs_ctx* c = (hs_ctx*)p;
  float* out = c->out;
  const float* tin = c->tin;
  const float* power = c->power;
  const int w = c->w, h = c->h;
  const float sdc = c->sdc, rx1 = c->rx1, ry1 = c->ry1, rz1 = c->rz1, amb = c->amb;
  for (int y = y0; y < y1; ++y) {
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const float t = tin[i];
      const float n = y > 0 ? tin[i - w] : t;
      const float s = y < h - 1 ? tin[i + w] : t;
      const float we = x > 0 ? tin[i - 1] : t;
      const float e = x < w - 1 ? tin[i + 1] : t;
      /* HS_STEP of kernels/hotspot.cu: explicit fmaf, same order */
      const float ns = fmaf(-2.0f, t, n + s);
      const float ew = fmaf(-2.0f, t, e + we);
      float d = fmaf(ns, ry1, power[i]);
      d = fmaf(ew, rx1, d);
      d = fmaf(amb - t, rz1, d);
      out[i] = fmaf(sdc, d, t);
    }
  }
}

static void hotspot_step(float* out, const float* tin, const float* power, int w, int h,
                         float sdc, float rx1, float ry1, float rz1, float amb) {
  hs_ctx c = {out, tin, power, w, h, sdc, rx1, ry1, rz1, amb};
  parallel_for(h, hotspot_rows, &c);
}

/* The tuned kernels' folded form (kernels/hotspot.cu header, HS_C/HS_FAST):
 * c = fmaf(ap, P, ac); T' = fmaf(ax, E+W, fmaf(ay, N+S, fmaf(at, T, c))). */
typedef struct {
  float* out;
  const float *tin, *power;
  int w, h;
  float at, ay, ax, ap, ac;
} hs_tuned_ctx;

static void hotspot_tuned_rows(void* p, int y0, int y1) {
  hs_tuned_ctx* c = (hs_tuned_ctx*)p;
  const float* tin = c->tin;
  const int w = c->w, h = c->h;
  for (int y = y0; y < y1; ++y) {
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const float t = tin[i];
      const float n = y > 0 ? tin[i - w] : t;
      const float s = y < h - 1 ? tin[i + w] : t;
      const float we = x > 0 ? tin[i - 1] : t;
      const float e = x < w - 1 ? tin[i + 1] : t;
      const float cp = fmaf(c->ap, c->power[i], c->ac);
      c->out[i] = fmaf(c->ax, e + we, fmaf(c->ay, n + s, fmaf(c->at, t, cp)));
    }
  }
}

void oracle_hotspot_tuned(float* out, const float* temp, const float* power, int w, int h,
                          int iterations, float at, float ay, float ax, float ap, float ac,
                          float* scratch) {
  const float* src = temp;
  for (int it = 0; it < iterations; ++it) {
    float* dst = ((iterations - 1 - it) % 2 == 0) ? out : scratch;
    hs_tuned_ctx c = {dst, src, power, w, h, at, ay, ax, ap, ac};
    parallel_for(h, hotspot_tuned_rows, &c);
    src = dst;
  }
  if (iterations == 0) memcpy(out, temp, sizeof(float) * (size_t)w * h);
}

/* `iterations` steps from `temp`; result in `out`; `scratch` is w*h floats. */
void oracle_hotspot(float* out, const float* temp, const float* power, int w, int h,
                    int iterations, float sdc, float rx1, float ry1, float rz1, float amb,
                    float* scratch) {
  const float* src = temp;
  for (int it = 0; it < iterations; ++it) {
    float* dst = ((iterations - 1 - it) % 2 == 0) ? out : scratch;
    hotspot_step(dst, src, power, w, h, sdc, rx1, ry1, rz1, amb);
    src = dst;
  }
  if (iterations == 0) memcpy(out, temp, sizeof(float) * (size_t)w * h);
}

/* out[dm][s] = sum_ch in[ch*pitch + s + trunc(dmv*delay[ch])], ascending ch,
 * dmv = dm_first + (float)dm * dm_step with explicit fp32 roundings
 * (kernels/dedispersion.cu). */
typedef struct {
  float* out;
  const float *in, *delay;
  int pitch, nch, nsamp;
  float dm_first, dm_step;
} dd_ctx;

static void dedisp_rows(void* p, int d0, int d1) {
  dd_ctx* c = (dd_ctx*)p;
  float* out = c->out;
  const float* in = c->in;
  const float* delay = c->delay;
  const int pitch = c->pitch, nch = c->nch, nsamp = c->nsamp;
  const float dm_first = c->dm_first, dm_step = c->dm_step;
  for (int dm = d0; dm < d1; ++dm) {
    volatile float prod = (float)dm * dm_step; /* force the fp32 rounding */
    const float dmv = dm_first + prod;
    int* sh = (int*)malloc(sizeof(int) * (size_t)nch);
    for (int ch = 0; ch < nch; ++ch) {
      volatile float p = dmv * delay[ch];
      sh[ch] = (int)truncf(p);
    }
    float* o = out + (size_t)dm * nsamp;
    for (int s = 0; s < nsamp; ++s) o[s] = 0.f;
    for (int ch = 0; ch < nch; ++ch) {
      const float* row = in + (size_t)ch * pitch + sh[ch];
      for (int s = 0; s < nsamp; ++s) o[s] = o[s] + row[s];
    }
    free(sh);
  }
}

void oracle_dedispersion(float* out, const float* in, int pitch, const float* delay, int nch,
                         int nsamp, int ndm, float dm_first, float dm_step) {
  dd_ctx c = {out, in, delay, pitch, nch, nsamp, dm_first, dm_step};
  parallel_for(ndm, dedisp_rows, &c);
}

/* c(m,n) = sum_k a(m,k) b(k,n) as one fmaf chain over ascending k;
 * a(m,k) = A[k*M+m], b(k,n) = B[k*N+n], c(m,n) = C[n*M+m]
 * (kernels/gemm.cu, CLBlast column-major view). */
typedef struct {
  float* c;
  const float *a, *b;
  int m, n, k;
} gemm_ctx;

static void gemm_cols(void* p, int j0, int j1) {
  gemm_ctx* g = (gemm_ctx*)p;
  float* c = g->c;
  const float* a = g->a;
  const float* b = g->b;
  const int m = g->m, n = g->n, k = g->k;
  for (int j = j0; j < j1; ++j) {
    float* col = c + (size_t)j * m;
    for (int i = 0; i < m; ++i) col[i] = 0.f;
    for (int kk = 0; kk < k; ++kk) {
      const float bv = b[(size_t)kk * n + j];
      const float* arow = a + (size_t)kk * m;
      for (int i = 0; i < m; ++i) col[i] = fmaf(arow[i], bv, col[i]);
    }
  }
}

void oracle_gemm(float* c, const float* a, const float* b, int m, int n, int k) {
  gemm_ctx g = {c, a, b, m, n, k};
  parallel_for(n, gemm_cols, &g);
}
