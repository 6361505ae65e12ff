// FP32 SIMT peak probe (roofline denominator for the FFMA-bound kernels).
// 16 independent FFMA chains per thread, full occupancy; FLOP = 2 * FMA.
extern "C" __global__ void __launch_bounds__(256) ffma_peak(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = (threadIdx.x + j) * 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  if (s == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Packed variant: fma.rn.f32x2 (FFMA2, sm_100+), 16 independent pairs.
extern "C" __global__ void __launch_bounds__(256) ffma2_peak(float* out, int iters, float a, float b) {
  unsigned long long x[16];
  const unsigned long long av = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  const unsigned long long bv = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float v = (threadIdx.x + j) * 1e-7f;
    x[j] = ((unsigned long long)__float_as_uint(v) << 32) | __float_as_uint(v + 1e-7f);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[j]) : "l"(av), "l"(bv));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += __uint_as_float((unsigned)x[j]) + __uint_as_float((unsigned)(x[j] >> 32));
  if (s == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
