// TF32 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// the north_star's optional B200 variant of the CLBlast GEMM.  Same
// product and output layout as kernels/gemm.cu, but the operands are held
// K-major in HBM (the layout the tf32 UMMA consumes; MN-major tf32
// operands read as zero on sm_100 -- measured, tools/cuda/mma_probe.cu):
//
//   a(m,k) = Ak[m*GK + k]   b(k,n) = Bk[n*GK + k]   c(m,n) = C[n*GM + m]
//
// One CTA computes a BM x BN = 128 x BN_T tile (BN_T in {128, 256}):
//   warp 0      TMA producer: per k-block of BK=32 one A box (32 K x 128 M)
//               and one B box (32 K x BN_T N), 128B swizzle (K-major
//               canonical: 128-B rows, 8-row / 1 KB atoms), into a
//               STAGES-deep ring guarded by full/empty mbarriers
//   warp 1      TMEM allocator + single-thread MMA issuer:
//               tcgen05.mma.cta_group::1.kind::tf32, M=128, N=BN_T, K=8,
//               4 per k-block, accumulator in TMEM (BN_T fp32 columns);
//               tcgen05.commit frees the smem stage / signals the epilogue
//   warps 2-5   epilogue: tcgen05.ld 32x32b (TMEM lane = m) -> registers
//               -> coalesced column stores of C (m contiguous)
// CLUSTER == 2: a 2-CTA thread-block cluster shares the B tile -- the two
// CTAs own consecutive M tiles of the same N tile; each TMA-loads its own
// A box and HALF of the B box, multicast into both CTAs' stage buffers
// (cp.async.bulk.tensor ... .multicast::cluster), so L2->SM operand traffic
// per output drops from (128+BN_T) to (128+BN_T/2) rows per k-block (the
// single-CTA kernel is bound by it: ~18 TB/s of TMA reads, ncu
// profiles/round2/ncu/ncu_gemm_tc_256-2.md).  A stage may be refilled only
// when BOTH CTAs' MMAs have consumed it: every MMA commit arrives on the
// empty barrier of both CTAs (tcgen05.commit ... .multicast::cluster), whose
// count is 2.
// Tunables (compile-time): BN_T, STAGES, CLUSTER.  Problem macros: GM, GN, GK.
// Precision: operands are read as TF32 (10-bit mantissa) by the tensor
// core, accumulation is fp32; verification uses a K-scaled tolerance.

#ifndef BN_T
#define BN_T 256
#endif
#ifndef STAGES
#define STAGES 4
#endif
#ifndef CLUSTER
#define CLUSTER 1
#endif
#define BM 128
#define BK 32
#define KSTEP 8
#define A_STAGE_BYTES (BM * BK * 4)
#define B_STAGE_BYTES (BN_T * BK * 4)
#define STAGE_BYTES (A_STAGE_BYTES + B_STAGE_BYTES)
#define NUM_THREADS 192
#define TMEM_COLS BN_T

struct __align__(64) TmaDesc {
  unsigned long long v[16];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(unsigned dst, const TmaDesc* desc, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(desc)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, 128B swizzle: rows of 128 B
// (32 tf32), 8-row atoms of 1 KB, SBO = 1024 (next 8 MN rows), LBO unused (16)
__device__ __forceinline__ unsigned long long umma_desc(unsigned addr, unsigned lbo, unsigned sbo) {
  unsigned long long d = 0;
  d |= (unsigned long long)((addr >> 4) & 0x3FFF);
  d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (Blackwell)
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// instruction descriptor: D=f32, A=B=tf32, A and B K-major, N=BN_T, M=128
#ifndef MAJOR_BITS
#define MAJOR_BITS 0u
#endif
#define IDESC_BASE ((1u << 4) | (2u << 7) | (2u << 10) | MAJOR_BITS | ((unsigned)(BM >> 4) << 24))
#define IDESC_N(n) (IDESC_BASE | ((unsigned)((n) >> 3) << 17))

__device__ __forceinline__ void umma_tf32(unsigned tmem_d, unsigned long long da, unsigned long long db,
                                          unsigned idesc, unsigned accumulate) {
#ifdef MMA_WITH_MASK
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
#endif
}

__device__ __forceinline__ void umma_commit(unsigned bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// commit arriving on the barrier at the same smem offset in every CTA of `mask`
__device__ __forceinline__ void umma_commit_mc(unsigned bar, unsigned short mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"(mask)
               : "memory");
}

// TMA 2-D load multicast into the same smem offset of every CTA in `mask`;
// each destination CTA's mbarrier (same offset) receives the byte count
__device__ __forceinline__ void tma_load_2d_mc(unsigned dst, const TmaDesc* desc, int c0, int c1, unsigned bar,
                                               unsigned short mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(desc)), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
      : "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

extern "C" __global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_tc_kernel(float* __restrict__ C, const __grid_constant__ TmaDesc tma_a,
               const __grid_constant__ TmaDesc tma_b, int tiles_m, int n_full) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms
  const unsigned base = smem_u32(smem_raw);
  const unsigned pad = (1024u - (base & 1023u)) & 1023u;
  unsigned char* smem = smem_raw + pad;
  const unsigned sbase = base + pad;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + STAGES * STAGE_BYTES);
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 2 * STAGES + 1);
  const unsigned full0 = smem_u32(bars);
  const unsigned empty0 = full0 + 8 * STAGES;
  const unsigned tfull = full0 + 16 * STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Work items (1-D grid): the first n_full are whole BM x BN_T tiles; the
  // tiles after them (which would form a partial last wave over the SMs)
  // are split into two BM x BN_T/2 halves each, so the last wave is as full
  // as the others (512 whole tiles on 148 SMs would cap at 86.5%).  A half
  // tile still TMA-loads a full BN_T-row B box (rows past its own 128 are
  // unused / zero-filled past GN) and runs the MMA with N = BN_T/2.
#if CLUSTER == 2
  // a cluster owns M tiles (2p, 2p+1) of one N tile; whole tiles only
  const unsigned crank = cluster_rank();
  const int pair = blockIdx.x >> 1;
  const int pairs_m = tiles_m >> 1;
  const int m0 = ((pair % pairs_m) * 2 + (int)crank) * BM;
  const int bn = BN_T;
  const int n0 = (pair / pairs_m) * BN_T;
  (void)n_full;
#else
  const int item = blockIdx.x;
  const int tile = item < n_full ? item : n_full + ((item - n_full) >> 1);
  const int half = item < n_full ? -1 : ((item - n_full) & 1);
  const int m0 = (tile % tiles_m) * BM;
  const int bn = half < 0 ? BN_T : BN_T / 2;
  const int n0 = (tile / tiles_m) * BN_T + (half > 0 ? BN_T / 2 : 0);
#endif
  const unsigned idesc = IDESC_N(bn);
  constexpr int KB = GK / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, CLUSTER);  // every CTA of the cluster releases the stage
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tma_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
#if CLUSTER == 2
  cluster_sync_all();  // the peer's barriers are initialised before anything targets them
#endif
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES;
        const unsigned ph = (kb / STAGES) & 1;
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        const unsigned full = full0 + 8 * s;
        mbar_expect_tx(full, STAGE_BYTES);
        const unsigned sa = sbase + s * STAGE_BYTES;
        const unsigned sb = sa + A_STAGE_BYTES;
        tma_load_2d(sa, &tma_a, kb * BK, m0, full);  // coords: (k, m)
#if CLUSTER == 2
        // this CTA's half of the B box, into both CTAs (same offset)
        tma_load_2d_mc(sb + crank * (B_STAGE_BYTES / 2), &tma_b, kb * BK, n0 + (int)crank * (BN_T / 2), full,
                       (unsigned short)0x3);
#else
        tma_load_2d(sb, &tma_b, kb * BK, n0, full);  // coords: (k, n)
#endif
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (single thread)
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES;
        const unsigned ph = (kb / STAGES) & 1;
        mbar_wait(full0 + 8 * s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
#ifdef DEBUG_DUMP_SMEM
        if (kb == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
          const unsigned* w = reinterpret_cast<const unsigned*>(smem);
          for (int i = 0; i < STAGE_BYTES / 4; ++i) reinterpret_cast<unsigned*>(C)[i] = w[i];
        }
#endif
        const unsigned sa = sbase + s * STAGE_BYTES;
        const unsigned sb = sa + A_STAGE_BYTES;
#pragma unroll
        for (int k = 0; k < BK / KSTEP; ++k) {
          // K step of 8 tf32 = 32 bytes along the swizzled 128-byte rows
          const unsigned long long da = umma_desc(sa + k * 32, 16, 1024);
          const unsigned long long db = umma_desc(sb + k * 32, 16, 1024);
#ifndef NO_MMA
          umma_tf32(tmem, da, db, idesc, (kb | k) != 0);
#else
          (void)da;
          (void)db;
#endif
        }
#if CLUSTER == 2
        umma_commit_mc(empty0 + 8 * s, (unsigned short)0x3);  // releases the stage in both CTAs
#else
        umma_commit(empty0 + 8 * s);  // frees the stage once these MMAs retire
#endif
      }
      umma_commit(tfull);  // accumulator complete
    }
  } else {
    // ---- epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
#ifdef DEBUG_TMEM_ST
    {  // write a known pattern into TMEM, skip waiting for the MMAs
      const unsigned ta = tmem + ((unsigned)(q * 32) << 16);
      for (int c = 0; c < BN_T; ++c) {
        unsigned val = __float_as_uint((float)((q * 32 + lane) * 1000 + c));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c), "r"(val));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
#else
    mbar_wait(tfull, 0);
#endif
    asm volatile("tcgen05.fence::after_thread_sync;");
#ifdef DEBUG_TMEM_ADDR
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 64) {
      C[0] = __uint_as_float(tmem);
    }
    if (blockIdx.x == 0 && blockIdx.y == 0) return;
#endif
    const int m = m0 + q * 32 + lane;
    const unsigned taddr = tmem + ((unsigned)(q * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < bn; c += 16) {
      unsigned r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#ifndef DEBUG_DUMP_SMEM
#pragma unroll
      for (int j = 0; j < 16; ++j) C[(size_t)(n0 + c + j) * GM + m] = __uint_as_float(r[j]);
#endif
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
#if CLUSTER == 2
  cluster_sync_all();  // no peer multicast or commit may still target this CTA's smem
#endif
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// smem bytes the host must request
#define GEMM_TC_SMEM (STAGES * STAGE_BYTES + 1024 + 256)
