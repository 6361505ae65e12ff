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

// TF32 tensor-pipe peak probe (denominator of the tcgen05 GEMM's roofline):
// per CTA one elected thread issues `iters` x 4 back-to-back
// tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=256, K=8, accumulator in
// TMEM) on operands resident in shared memory -- no loads, no epilogue, the
// tensor pipe alone.  One commit at the end; FLOP = 2*128*256*8 per MMA.
// Operand contents are irrelevant (zeros), the instruction shape is what
// the GEMM issues (K-major, 128B swizzle descriptors).
#define PK_BN 256
__device__ __forceinline__ unsigned pk_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned long long pk_desc(unsigned addr) {
  unsigned long long d = 0;
  d |= (unsigned long long)((addr >> 4) & 0x3FFF);
  d |= (unsigned long long)(1u) << 16;         // LBO 16 B (unused with swizzle)
  d |= (unsigned long long)(1024u >> 4) << 32;  // SBO: next 8-row atom
  d |= 1ull << 46;
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}
extern "C" __global__ void __launch_bounds__(128, 1) tf32_mma_peak(float* out, int iters) {
  extern __shared__ unsigned char pk_raw[];
  const unsigned base = pk_smem_u32(pk_raw);
  const unsigned pad = (1024u - (base & 1023u)) & 1023u;
  unsigned char* sm = pk_raw + pad;
  const unsigned sa = base + pad, sb = sa + 128 * 128;  // A: 128 rows x 128 B, B: 256 rows x 128 B
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + 128 * 128 + PK_BN * 128);
  unsigned* slot = reinterpret_cast<unsigned*>(bar + 1);
  for (int i = threadIdx.x; i < (128 * 128 + PK_BN * 128) / 4; i += blockDim.x)
    reinterpret_cast<unsigned*>(sm)[i] = 0u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(pk_smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(pk_smem_u32(slot)),
                 "r"(PK_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = *slot;
  const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(PK_BN >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned long long da = pk_desc(sa + k * 32), db = pk_desc(sb + k * 32);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"((unsigned)(it | k)));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(pk_smem_u32(bar))
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
          pk_smem_u32(bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    unsigned r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (__uint_as_float(r) == 1234.5f) out[blockIdx.x] = 1.f;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(PK_BN));
  }
}
