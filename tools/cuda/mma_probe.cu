// Minimal tcgen05.mma probe: A, B = 1.0 in smem (written by threads), one
// M=128 N=128 K=8 tf32 MMA, D read back.  Expect D = 8 everywhere.
// variant bit 0: MN-major (else K-major); bit 1: 128B swizzle (else none)
// variant bit 2: use lbo/sbo swapped
__device__ __forceinline__ unsigned long long desc(unsigned addr, unsigned lbo, unsigned sbo, unsigned layout) {
  unsigned long long d = 0;
  d |= (unsigned long long)((addr >> 4) & 0x3FFF);
  d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= (unsigned long long)layout << 61;
  return d;
}

extern "C" __global__ void __launch_bounds__(128, 1) mma_probe(float* out, int variant, unsigned lbo, unsigned sbo) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned slot;
  __shared__ __align__(8) unsigned long long bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* fs = reinterpret_cast<float*>(sm);
  for (int i = threadIdx.x; i < 2 * 128 * 8 + 4096; i += 128) fs[i] = 1.0f;  // A (4KB) + B (4KB) + slack
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = slot;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const bool mn = variant & 1;
  const unsigned layout = (variant & 2) ? 2u : 0u;
  const unsigned majors = mn ? ((1u << 15) | (1u << 16)) : 0u;
  const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | majors | (16u << 17) | (8u << 24);
  if (threadIdx.x == 0) {
    const unsigned long long da = desc(base, lbo, sbo, layout);
    const unsigned long long db = desc(base + 8192, lbo, sbo, layout);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (unsigned)__cvta_generic_to_shared(&bar)) : "memory");
  }
  {
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            (unsigned)__cvta_generic_to_shared(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  unsigned r[4];
  const unsigned ta = tmem + ((unsigned)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 4; ++j) out[threadIdx.x * 4 + j] = __uint_as_float(r[j]);
  if (threadIdx.x == 0) out[600] = __uint_as_float(base);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}
