// TF32 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// the north_star's optional B200 variant of the CLBlast GEMM.  Same
// product and output layout as kernels/gemm.cu, but the operands are held
// K-major in HBM (the layout the tf32 UMMA consumes; MN-major tf32
// operands read as zero on sm_100 -- measured, tools/cuda/mma_probe.cu):
//
//   a(m,k) = Ak[m*GK + k]   b(k,n) = Bk[n*GK + k]   c(m,n) = C[n*GM + m]
//
// PERSISTENT kernel: one CTA per SM (or one 2-CTA cluster per SM pair)
// loops over work items -- 128 x BN_T output tiles (BN_T in {128, 256}),
// and, for the tiles that would form a partial last wave, half tiles of
// 128 x BN_T/2 -- assigned round-robin (item = cta + i * ncta).  Warp roles:
//   warp 0      TMA producer: per k-block of BK=32 one A box (32 K x 128 M)
//               and one B box (32 K x BN_T N), 128B swizzle (K-major
//               canonical: 128-B rows, 8-row / 1 KB atoms), into a
//               STAGES-deep ring guarded by full/empty mbarriers; it runs
//               straight on into the next item's k-blocks
//   warp 1      TMEM allocator + single-thread MMA issuer:
//               tcgen05.mma.cta_group::1.kind::tf32, M=128, N=BN_T, K=8,
//               4 per k-block, into one of TWO TMEM accumulators (2 x BN_T
//               fp32 columns): item i accumulates in buffer i & 1 while the
//               epilogue drains buffer (i-1) & 1 -- the tensor pipe never
//               waits for an epilogue; tcgen05.commit frees smem stages and
//               signals "accumulator full"
//   warps 2-5   epilogue: tcgen05.ld 32x32b (TMEM lane = m) -> registers
//               -> coalesced column stores of C (m contiguous), then one
//               arrival per warp on the buffer's "accumulator empty" barrier
// CLUSTER == 2: a 2-CTA thread-block cluster shares the B tile -- the two
// CTAs own consecutive M tiles of the same N tile; each TMA-loads its own
// A box and HALF of the B box, multicast into both CTAs' stage buffers
// (cp.async.bulk.tensor ... .multicast::cluster), so L2->SM operand traffic
// per output drops from (128+BN_T) to (128+BN_T/2) rows per k-block.  A
// stage may be refilled only when BOTH CTAs' MMAs have consumed it: every
// MMA commit arrives on the empty barrier of both CTAs (tcgen05.commit ...
// .multicast::cluster), whose count is 2.  Both CTAs of a cluster walk the
// same item sequence, so their k-block counters stay in lock step.
// CLUSTER == 4: a 2 x 2 cluster owns 2 M tiles x 2 N tiles; CTA rank r is
// (rm, rn) = (r & 1, r >> 1).  The two CTAs of an M tile each load half of
// its A box and multicast it to both; the two CTAs of an N tile do the same
// with B -- per CTA (64 + BN_T/2) rows per k-block instead of 128 + BN_T.
// Every MMA commit arrives on the empty barrier of all four CTAs (count 4):
// a stage is refilled only when every CTA that receives data into it has
// consumed it.
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
#define TMEM_COLS (2 * BN_T)  // two accumulators

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

// work item -> this CTA's output origin (m0, n0); see the kernel comment
__device__ __forceinline__ void gemm_tc_item(int item, int n_full, int tiles_m, unsigned crank, int& m0, int& n0) {
  const int tile = item < n_full ? item : n_full + ((item - n_full) >> 1);
  const int half = item < n_full ? 0 : ((item - n_full) & 1);
#if CLUSTER == 4
  const int pairs_m = tiles_m >> 1;  // a cluster owns M tiles (2pm, 2pm+1) x N tiles (2pn, 2pn+1)
  m0 = ((tile % pairs_m) * 2 + (int)(crank & 1)) * BM;
  n0 = ((tile / pairs_m) * 2 + (int)(crank >> 1)) * BN_T + half * (BN_T / 2);
#elif CLUSTER == 2
  const int pairs_m = tiles_m >> 1;  // a cluster owns M tiles (2p, 2p+1) of one N tile
  m0 = ((tile % pairs_m) * 2 + (int)crank) * BM;
  n0 = (tile / pairs_m) * BN_T + half * (BN_T / 2);
#else
  (void)crank;
  m0 = (tile % tiles_m) * BM;
  n0 = (tile / tiles_m) * BN_T + half * (BN_T / 2);
#endif
}

extern "C" __global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_tc_kernel(float* __restrict__ C, const __grid_constant__ TmaDesc tma_a,
               const __grid_constant__ TmaDesc tma_b, int tiles_m, int n_full, int n_items) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms
  const unsigned base = smem_u32(smem_raw);
  const unsigned pad = (1024u - (base & 1023u)) & 1023u;
  const unsigned sbase = base + pad;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw + pad + STAGES * STAGE_BYTES);
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 2 * STAGES + 4);
  const unsigned full0 = smem_u32(bars);
  const unsigned empty0 = full0 + 8 * STAGES;
  const unsigned tfull0 = full0 + 16 * STAGES;   // accumulator full [2]
  const unsigned tempty0 = tfull0 + 16;          // accumulator empty [2]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // work-item walk: CTA (CLUSTER == 1) or cluster (CLUSTER == 2) `unit`
  // takes items unit, unit + nunits, ...  Items < n_full are whole tiles
  // (pairs of M tiles for CLUSTER == 2), the rest halves of the remaining
  // tiles along N (a half still loads a full B box; rows past it unused).
#if CLUSTER > 1
  const unsigned crank = cluster_rank();
  const int unit = blockIdx.x / CLUSTER;
  const int nunits = gridDim.x / CLUSTER;
#else
  const unsigned crank = 0;
  const int unit = blockIdx.x;
  const int nunits = gridDim.x;
#endif
  constexpr int KB = GK / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, CLUSTER);  // every CTA of the cluster releases the stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, 1);   // MMA commit
      mbar_init(tempty0 + 8 * b, 4);  // one arrival per epilogue warp
    }
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
#if CLUSTER > 1
  cluster_sync_all();  // the peers' barriers are initialised before anything targets them
#endif
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int g = 0;  // k-blocks issued so far (stage / phase)
      for (int item = unit; item < n_items; item += nunits) {
        int m0, n0;
        gemm_tc_item(item, n_full, tiles_m, crank, m0, n0);
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % STAGES;
          mbar_wait(empty0 + 8 * s, ((g / STAGES) & 1) ^ 1);
          const unsigned full = full0 + 8 * s;
          mbar_expect_tx(full, STAGE_BYTES);
          const unsigned sa = sbase + s * STAGE_BYTES;
          const unsigned sb = sa + A_STAGE_BYTES;
#if CLUSTER == 4
          {  // half of the A box to the M-tile's two CTAs, half of the B box to the N-tile's two
            const unsigned rm = crank & 1, rn = crank >> 1;
            tma_load_2d_mc(sa + rn * (A_STAGE_BYTES / 2), &tma_a, kb * BK, m0 + (int)rn * (BM / 2), full,
                           (unsigned short)((1u << rm) | (1u << (rm + 2))));
            tma_load_2d_mc(sb + rm * (B_STAGE_BYTES / 2), &tma_b, kb * BK, n0 + (int)rm * (BN_T / 2), full,
                           (unsigned short)(3u << (2 * rn)));
          }
#elif CLUSTER == 2
          tma_load_2d(sa, &tma_a, kb * BK, m0, full);  // coords: (k, m)
          // this CTA's half of the B box, into both CTAs (same offset)
          tma_load_2d_mc(sb + crank * (B_STAGE_BYTES / 2), &tma_b, kb * BK, n0 + (int)crank * (BN_T / 2), full,
                         (unsigned short)0x3);
#else
          tma_load_2d(sa, &tma_a, kb * BK, m0, full);  // coords: (k, m)
          tma_load_2d(sb, &tma_b, kb * BK, n0, full);  // coords: (k, n)
#endif
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (single thread)
      int g = 0, it = 0;
      for (int item = unit; item < n_items; item += nunits, ++it) {
        const int buf = it & 1;
        const unsigned idesc = IDESC_N(item < n_full ? BN_T : BN_T / 2);
        const unsigned acc = tmem + (unsigned)(buf * BN_T);
        mbar_wait(tempty0 + 8 * buf, ((it >> 1) & 1) ^ 1);  // epilogue drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % STAGES;
          mbar_wait(full0 + 8 * s, (g / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const unsigned sa = sbase + s * STAGE_BYTES;
          const unsigned sb = sa + A_STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / KSTEP; ++k) {
            // K step of 8 tf32 = 32 bytes along the swizzled 128-byte rows
            const unsigned long long da = umma_desc(sa + k * 32, 16, 1024);
            const unsigned long long db = umma_desc(sb + k * 32, 16, 1024);
            umma_tf32(acc, da, db, idesc, (kb | k) != 0);
          }
#if CLUSTER > 1
          umma_commit_mc(empty0 + 8 * s, (unsigned short)((1u << CLUSTER) - 1));  // releases the stage in every CTA
#else
          umma_commit(empty0 + 8 * s);  // frees the stage once these MMAs retire
#endif
        }
        umma_commit(tfull0 + 8 * buf);  // accumulator complete
      }
    }
  } else {
    // ---- epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
    int it = 0;
    for (int item = unit; item < n_items; item += nunits, ++it) {
      const int buf = it & 1;
      int m0, n0;
      gemm_tc_item(item, n_full, tiles_m, crank, m0, n0);
      const int bn = item < n_full ? BN_T : BN_T / 2;
      mbar_wait(tfull0 + 8 * buf, (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int m = m0 + q * 32 + lane;
      const unsigned taddr = tmem + ((unsigned)(q * 32) << 16) + (unsigned)(buf * BN_T);
#pragma unroll 1
      for (int c = 0; c < bn; c += 16) {
        unsigned r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) C[(size_t)(n0 + c + j) * GM + m] = __uint_as_float(r[j]);
      }
      // this warp's TMEM reads are complete: hand the buffer back to the MMA issuer
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty0 + 8 * buf) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
#if CLUSTER > 1
  cluster_sync_all();  // no peer multicast or commit may still target this CTA's smem
#endif
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// smem bytes the host must request
#define GEMM_TC_SMEM (STAGES * STAGE_BYTES + 1024 + 256)
