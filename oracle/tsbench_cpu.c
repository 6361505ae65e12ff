/*
 * oracle/tsbench_cpu.c -- the CPU benchmark PROGRAM the reference drives.
 *
 * BASELINE INFRASTRUCTURE ONLY (never the product path).  The reference's
 * only executor runs a benchmark program per configuration and reads its
 * stdout (`ts/measure.py:218-305`: one `TUNE_TIME_MS <ms>` line per run; a
 * program printing several lines in one launch is "self-reporting" and its
 * last `benchmark_runs` values count).  bench.py's reference arm runs the
 * UNMODIFIED reference (installed under baseline/_ref) with
 *   --backend 'cmd:oracle/tsbench_cpu hotspot --threads N --runs 8 {block_size_x} ...'
 * so the reference's own CPU path -- its tuning loop, process protocol and
 * parsing -- times the C oracle kernel (kernels.c, all host threads) on the
 * full BASELINE size.  GPU tunables do not change CPU arithmetic; they are
 * accepted (for the command template) and ignored.
 *
 *   tsbench_cpu hotspot|convolution|gemm [--w W] [--h H] [--iters I]
 *               [--threads N] [--runs R] [config values ...]
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

void oracle_set_threads(int n);
void oracle_hotspot(float* out, const float* temp, const float* power, int w, int h, int iterations,
                    float sdc, float rx1, float ry1, float rz1, float amb, float* scratch);
void oracle_convolution(float* out, const float* in, int pitch, int w, int h, const float* f, int fw,
                        int fh);
void oracle_gemm(float* c, const float* a, const float* b, int m, int n, int k);

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static float* filled(size_t n, unsigned seed, float lo, float span) {
  float* p = (float*)malloc(n * sizeof(float));
  if (!p) {
    fprintf(stderr, "out of memory\n");
    exit(3);
  }
  unsigned x = seed * 2654435761u + 1u;
  for (size_t i = 0; i < n; ++i) {
    x = x * 1664525u + 1013904223u;
    p[i] = lo + span * (float)(x >> 8) * (1.0f / 16777216.0f);
  }
  return p;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s hotspot|convolution|gemm [--w W] [--h H] [--iters I] [--threads N] [--runs R]\n",
            argv[0]);
    puts("TUNE_STATUS invalid");
    return 2;
  }
  const char* kernel = argv[1];
  int w = 4096, h = 4096, iters = 20, threads = 0, runs = 8;
  for (int i = 2; i + 1 < argc; ++i) {
    if (!strcmp(argv[i], "--w")) w = atoi(argv[++i]);
    else if (!strcmp(argv[i], "--h")) h = atoi(argv[++i]);
    else if (!strcmp(argv[i], "--iters")) iters = atoi(argv[++i]);
    else if (!strcmp(argv[i], "--threads")) threads = atoi(argv[++i]);
    else if (!strcmp(argv[i], "--runs")) runs = atoi(argv[++i]);
  }
  if (threads > 0) oracle_set_threads(threads);
  size_t n = (size_t)w * h;
  if (!strcmp(kernel, "hotspot")) {
    float* temp = filled(n, 3, 323.15f, 10.0f);
    float* power = filled(n, 4, 0.0f, 1e-3f);
    float* out = filled(n, 5, 0.0f, 0.0f);
    float* scratch = filled(n, 6, 0.0f, 0.0f);
    /* Rodinia chip constants at 4096^2 with the 512^2 cell size (problems.Hotspot) */
    const float sdc = 0.0178574f, rx1 = 0.05f, ry1 = 0.05f, rz1 = 0.0016f, amb = 80.0f;
    for (int r = 0; r < runs; ++r) {
      double t0 = now_ms();
      oracle_hotspot(out, temp, power, w, h, iters, sdc, rx1, ry1, rz1, amb, scratch);
      printf("TUNE_TIME_MS %.6f\n", now_ms() - t0);
      fflush(stdout);
    }
  } else if (!strcmp(kernel, "convolution")) {
    const int fw = 15, pitch = w + fw - 1;
    float* in = filled((size_t)pitch * (h + fw - 1), 1, 0.0f, 1.0f);
    float* f = filled((size_t)fw * fw, 2, 0.0f, 1.0f);
    float* out = filled(n, 7, 0.0f, 0.0f);
    for (int r = 0; r < runs; ++r) {
      double t0 = now_ms();
      oracle_convolution(out, in, pitch, w, h, f, fw, fw);
      printf("TUNE_TIME_MS %.6f\n", now_ms() - t0);
      fflush(stdout);
    }
  } else if (!strcmp(kernel, "gemm")) {
    float* a = filled(n, 6, -1.0f, 2.0f);
    float* b = filled(n, 7, -1.0f, 2.0f);
    float* c = filled(n, 8, 0.0f, 0.0f);
    for (int r = 0; r < runs; ++r) {
      double t0 = now_ms();
      oracle_gemm(c, a, b, w, h, w);
      printf("TUNE_TIME_MS %.6f\n", now_ms() - t0);
      fflush(stdout);
    }
  } else {
    puts("TUNE_STATUS invalid");
    return 2;
  }
  return 0;
}
