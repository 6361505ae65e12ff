// TF32 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// the north_star's optional B200 variant of the CLBlast GEMM.  Same
// product and output layout as kernels/gemm.cu, but the operands are held
// K-major in HBM (the layout the tf32 UMMA consumes; MN-major tf32
// operands read as zero on sm_100 -- measured, tools/cuda/mma_probe.cu):
//
//   a(m,k) = Ak[m*GK + k]   b(k,n) = Bk[n*GK + k]   c(m,n) = C[n*GM + m]
//
// PERSISTENT kernel: one CTA per SM (CLUSTER == 1) or one CTA PAIR per two
// SMs (CLUSTER == 2) loops over work items -- output tiles of (128 *
// CLUSTER) x BN_T, and, for the tiles that would form a partial last wave,
// halves of BN_T/2 columns -- assigned round-robin (item = unit + i * nunits).
// Warp roles (per CTA):
//   warp 0      TMA producer: per k-block of BK=32 one A box (32 K x 128 M)
//               and one B box (32 K x BN_T/CLUSTER N), 128B swizzle (K-major
//               canonical: 128-B rows, 8-row / 1 KB atoms), into a
//               STAGES-deep ring guarded by full/empty mbarriers; it runs
//               straight on into the next item's k-blocks
//   warp 1      TMEM allocator + single-thread MMA issuer:
//               tcgen05.mma.kind::tf32, K=8, 4 per k-block, into one of TWO
//               TMEM accumulators (2 x BN_T fp32 columns): item i
//               accumulates in buffer i & 1 while the epilogue drains
//               buffer (i-1) & 1, so the tensor pipe never waits for an
//               epilogue; tcgen05.commit frees smem stages and signals
//               "accumulator full"
//   warps 2-5   epilogue: tcgen05.ld 32x32b (TMEM lane = m) -> registers
//               -> coalesced column stores of C (m contiguous), then one
//               arrival per warp on the buffer's "accumulator empty" barrier
//
// CLUSTER == 2 -- the 2-SM UMMA (cta_group::2): the pair computes a
// 256 x BN_T tile with ONE tcgen05.mma.cta_group::2 (M = 256) issued by the
// leader CTA; each CTA holds the A rows of its own 128-row half and HALF of
// the B tile (BN_T/2 rows), and the tensor cores of both SMs read both
// halves of B.  Per SM and k-block the smem traffic is A 16 KB + B BN_T/2
// rows instead of A + all BN_T rows: the single-CTA kernel needs ~178 B of
// smem traffic per cycle at the tensor peak (TMA writes + UMMA reads), over
// the 128 B/cycle an SM has; the pair needs ~117.  Protocol:
//   * both CTAs' TMA loads complete on the LEADER's full barrier (the
//     .cta_group::2 form of cp.async.bulk.tensor; address via mapa), armed
//     by the leader with the bytes of both CTAs;
//   * the leader's MMA commits arrive (multicast) on the empty barrier of
//     both CTAs -- each producer refills its own stage -- and on both
//     CTAs' accumulator-full barriers;
//   * all 8 epilogue warps of the pair arrive on the leader's
//     accumulator-empty barrier (remote mbarrier arrive).
// (A 2-CTA cluster that only multicast the B box, each CTA running its own
// 128-row MMA, and a 2 x 2 cluster multicasting halves of both boxes were
// measured round 2: no faster / 1.8x slower -- they cut L2 reads, not the
// per-SM smem traffic.)
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
#define B_ROWS (BN_T / CLUSTER)  // B rows held per CTA
#define B_STAGE_BYTES (B_ROWS * BK * 4)
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

// this CTA's shared address `a` as seen in CTA `rank` of the cluster
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__device__ __forceinline__ void tma_load_2d(unsigned dst, const TmaDesc* desc, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(desc)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// 2-SM form: data lands in THIS CTA's smem (`dst`), the byte count on the
// barrier `bar` (a shared::cluster address -- here the leader's)
__device__ __forceinline__ void tma_load_2d_pair(unsigned dst, const TmaDesc* desc, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
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

// instruction descriptor: D=f32, A=B=tf32, A and B K-major, M = 128 per CTA
// (256 for the pair), N = n
#define IDESC_BASE ((1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)((BM * CLUSTER) >> 4) << 24))
#define IDESC_N(n) (IDESC_BASE | ((unsigned)((n) >> 3) << 17))

__device__ __forceinline__ void umma_tf32(unsigned tmem_d, unsigned long long da, unsigned long long db,
                                          unsigned idesc, unsigned accumulate) {
#if CLUSTER == 2
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
#endif
}

// MMA completion -> mbarrier (CLUSTER == 2: the barrier at the same offset
// in both CTAs of the pair)
__device__ __forceinline__ void umma_commit(unsigned bar) {
#if CLUSTER == 2
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((unsigned short)0x3)
      : "memory");
#else
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
#endif
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// work item -> this CTA's output origin (m0, n0) and the item's N extent.
// Tiles are walked in BANDS of GEMM_BAND M units (all N tiles of a band,
// M fastest): the units in flight at once touch one band of A and at most
// a wave's worth of B, instead of all of A (64 MB) next to the C being
// written -- measured: all-M-first order re-read A from DRAM (343 MB read
// per launch against 128 MB compulsory)
#ifndef GEMM_BAND
#define GEMM_BAND 8
#endif
__device__ __forceinline__ void gemm_tc_item(int item, int n_full, int tiles_m, unsigned crank, int& m0, int& n0,
                                             int& bn) {
  const int tile = item < n_full ? item : n_full + ((item - n_full) >> 1);
  const int half = item < n_full ? 0 : ((item - n_full) & 1);
  const int units_m = tiles_m / CLUSTER;  // a pair owns M tiles (2p, 2p+1) of one N tile
  constexpr int tiles_n = GN / BN_T;
  const int band = (units_m % GEMM_BAND == 0) ? GEMM_BAND : units_m;
  const int per_band = band * tiles_n;
  const int r = tile % per_band;
  const int um = (tile / per_band) * band + r % band;
  const int un = r / band;
  m0 = (um * CLUSTER + (int)crank) * BM;
  n0 = un * BN_T + half * (BN_T / 2);
  bn = item < n_full ? BN_T : BN_T / 2;
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
  const unsigned tfull0 = full0 + 16 * STAGES;  // accumulator full [2]
  const unsigned tempty0 = tfull0 + 16;         // accumulator empty [2]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
#if CLUSTER == 2
  const unsigned crank = cluster_rank();
  const bool leader = crank == 0;
#else
  const unsigned crank = 0;
  const bool leader = true;
#endif
  const int unit = blockIdx.x / CLUSTER;
  const int nunits = gridDim.x / CLUSTER;
  constexpr int KB = GK / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);   // the (leader's) arming arrive + TMA bytes
      mbar_init(empty0 + 8 * s, 1);  // the (leader's) MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, 1);             // MMA commit
      mbar_init(tempty0 + 8 * b, 4 * CLUSTER);  // every epilogue warp of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tma_b)) : "memory");
  }
  if (warp == 1) {  // the same warp of both CTAs allocates (cta_group::2: jointly)
#if CLUSTER == 2
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
#else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
#endif
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
#if CLUSTER == 2
  cluster_sync_all();  // the peer's barriers are initialised before anything targets them
#endif
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs)
#if CLUSTER == 2
      const unsigned lfull0 = mapa(full0, 0);  // the leader's full barriers
#endif
      int g = 0;  // k-blocks issued so far (stage / phase)
      for (int item = unit; item < n_items; item += nunits) {
        int m0, n0, bn;
        gemm_tc_item(item, n_full, tiles_m, crank, m0, n0, bn);
        const int nb = n0 + (int)crank * (bn / CLUSTER);  // this CTA's B rows
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % STAGES;
          mbar_wait(empty0 + 8 * s, ((g / STAGES) & 1) ^ 1);
          const unsigned sa = sbase + s * STAGE_BYTES;
          const unsigned sb = sa + A_STAGE_BYTES;
#if CLUSTER == 2
          if (leader) mbar_expect_tx(full0 + 8 * s, 2 * STAGE_BYTES);  // both CTAs' bytes
          tma_load_2d_pair(sa, &tma_a, kb * BK, m0, lfull0 + 8 * s);
          tma_load_2d_pair(sb, &tma_b, kb * BK, nb, lfull0 + 8 * s);
#else
          mbar_expect_tx(full0 + 8 * s, STAGE_BYTES);
          tma_load_2d(sa, &tma_a, kb * BK, m0, full0 + 8 * s);  // coords: (k, m)
          tma_load_2d(sb, &tma_b, kb * BK, nb, full0 + 8 * s);  // coords: (k, n)
#endif
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---- MMA issuer (single thread of the leader)
      int g = 0, it = 0;
      for (int item = unit; item < n_items; item += nunits, ++it) {
        const int buf = it & 1;
        const unsigned idesc = IDESC_N(item < n_full ? BN_T : BN_T / 2);
        const unsigned acc = tmem + (unsigned)(buf * BN_T);
        mbar_wait(tempty0 + 8 * buf, ((it >> 1) & 1) ^ 1);  // every epilogue warp drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % STAGES;
          mbar_wait(full0 + 8 * s, (g / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const unsigned sa = sbase + s * STAGE_BYTES;
          const unsigned sb = sa + A_STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / KSTEP; ++k) {
            // K step of 8 tf32 = 32 bytes along the swizzled 128-byte rows;
            // for the pair the same offsets address the peer's halves
            const unsigned long long da = umma_desc(sa + k * 32, 16, 1024);
            const unsigned long long db = umma_desc(sb + k * 32, 16, 1024);
            umma_tf32(acc, da, db, idesc, (kb | k) != 0);
          }
          umma_commit(empty0 + 8 * s);  // frees the stage (in both CTAs) once these MMAs retire
        }
        umma_commit(tfull0 + 8 * buf);  // accumulator complete (in both CTAs)
      }
    }
  } else {
    // ---- epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
#if CLUSTER == 2
    const unsigned ltempty0 = mapa(tempty0, 0);  // the leader's accumulator-empty barriers
#else
    const unsigned ltempty0 = tempty0;
#endif
    int it = 0;
    for (int item = unit; item < n_items; item += nunits, ++it) {
      const int buf = it & 1;
      int m0, n0, bn;
      gemm_tc_item(item, n_full, tiles_m, crank, m0, n0, bn);
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
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ltempty0 + 8 * buf)
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
#if CLUSTER == 2
  cluster_sync_all();  // no peer TMA, commit or arrive may still target this CTA's smem
#endif
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
#if CLUSTER == 2
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
#else
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
#endif
  }
}

// smem bytes the host must request
#define GEMM_TC_SMEM (STAGES * STAGE_BYTES + 1024 + 256)
