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
