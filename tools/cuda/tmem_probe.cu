// Minimal TMEM round trip probe: alloc -> st pattern -> ld -> global.
extern "C" __global__ void __launch_bounds__(128, 1) tmem_probe(float* out, int variant) {
  __shared__ unsigned slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = slot;
  const unsigned ta = tmem + ((unsigned)(warp * 32) << 16);
  for (int c = 0; c < 32; ++c) {
    unsigned val = __float_as_uint((float)((warp * 32 + lane) * 100 + c));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c), "r"(val) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  unsigned r[4];
  if (variant == 0) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta + 4) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  } else {
    for (int j = 0; j < 4; ++j) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[j]) : "r"(ta + 4 + j) : "memory");
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
  for (int j = 0; j < 4; ++j) out[threadIdx.x * 4 + j] = __uint_as_float(r[j]);
  if (threadIdx.x == 0) out[512] = __uint_as_float(tmem);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}
