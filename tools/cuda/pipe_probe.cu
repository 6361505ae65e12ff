// FMA-pipe latency/throughput probe: C independent dependent chains per
// thread of scalar FFMA or packed FFMA2, W warps per SM (grid = #SMs).
#ifndef C
#define C 1
#endif
extern "C" __global__ void ffma_chain(float* out, int iters, float a, float b) {
  float x[C];
#pragma unroll
  for (int j = 0; j < C; ++j) x[j] = threadIdx.x * 1e-7f + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < C; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[j]) : "f"(a), "f"(b));
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < C; ++j) s += x[j];
  if (s == 1234.5f) out[threadIdx.x] = s;
}
extern "C" __global__ void ffma2_chain(float* out, int iters, float a, float b) {
  unsigned long long x[C];
  const unsigned long long av = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  const unsigned long long bv = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
#pragma unroll
  for (int j = 0; j < C; ++j) x[j] = (unsigned long long)(threadIdx.x + j);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < C; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[j]) : "l"(av), "l"(bv));
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < C; ++j) s += __uint_as_float((unsigned)x[j]);
  if (s == 1234.5f) out[threadIdx.x] = s;
}
