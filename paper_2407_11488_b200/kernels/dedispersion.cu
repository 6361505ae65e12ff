// Brute-force dedispersion, AMBER style (paper Table 1 dedispersion
// column; space paper_2407_11488_b200/spaces/dedispersion.spec == ref
// ts/spaces/dedispersion.spec:8-20).
//
//   out[dm][s] = sum_{ch < NCH} in[ch][s + shift(dm, ch)]
//   shift(dm, ch) = trunc( fp32( dmval(dm) * delay[ch] ) )
//   dmval(dm)     = fp32( dm_first + fp32( (float)dm * dm_step ) )
//
// All roundings are explicit (__fmul_rn / __fadd_rn) and channels are
// summed in ascending order, so every configuration, the reference
// kernel and the CPU oracle (oracle/kernels.c) agree bit-for-bit.
//
// x = samples, y = DMs.  Tunables:
//   BSX, BSY   thread block (samples x DMs)
//   TSX, TSY   samples / DMs per thread
//   STX, STY   tile_stride_x/y: 1 = a thread's samples (DMs) are strided
//              by the block size (coalesced across lanes), 0 = contiguous
// The input row of a channel is read through the read-only path; the
// per-channel delay lives in __constant__ (uniform across the warp).
// Grid: x = DM tiles (fastest), y = sample tiles, so the blocks sweeping
// one sample range for ALL DMs are co-resident and the 157 MB input is
// streamed from HBM ~once (L2 reuse) instead of once per DM-tile row.
// Problem macros: NCH, NSAMP, NDM, IN_PITCH.

__constant__ float d_delay[NCH];

#ifndef REFERENCE_ONLY

#define STR2(x) #x
#define STR(x) STR2(x)

#if (defined(DD_WIN) && DD_WIN) || (defined(DD_STG) && DD_STG)
// Shared-memory staging: per chunk of CC = 32 channels, each channel's
// block-wide row segment (the block's 32*TSX samples shifted by the block's
// FIRST DM, plus BLKSPAN + SPAN samples of DM spread, aligned down to 16 B)
// is brought in by one TMA bulk copy (cp.async.bulk, issued by warp 0's
// lanes, completion on the stage's mbarrier), NSTAGE chunks in flight.
// Warps then read their windows with LDS: 32 consecutive floats at any
// alignment are one conflict-free wavefront (an unaligned 128-byte global
// load costs ~2.4 L1 wavefronts and an LSU queue slot).
#define CC 32
#if defined(DD_WIN) && DD_WIN
#define ROWLEN ((32 * TSX + BLKSPAN + SPAN + 4 + 3) & ~3)
#else
#define ROWLEN ((BSX * TSX + BLKSPAN + 4 + 3) & ~3)
#endif
#ifndef DD_NSTAGE
#define DD_NSTAGE 5
#endif
#define NSTAGE DD_NSTAGE

__device__ __forceinline__ unsigned dd_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void dd_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(dd_smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void dd_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dd_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void dd_mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dd_smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void dd_mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(dd_smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void dd_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dd_smem_u32(dst)), "l"(src), "r"(bytes), "r"(dd_smem_u32(b))
      : "memory");
}

// warp 0: stage chunk t (channels t*CC ..) into `stage`
__device__ __forceinline__ void dd_issue_chunk(const float* __restrict__ in, float* stage, unsigned long long* bar,
                                               int t, int sb, float dmb, int lane, const float* sdelay) {
  const int ch = t * CC + lane;
  const int nvalid = NCH - t * CC < CC ? NCH - t * CC : CC;
  if (lane == 0) dd_mbar_expect(bar, (unsigned)(nvalid * ROWLEN * 4));
  __syncwarp();
  if (ch < NCH) {
    const int shb = __float2int_rz(__fmul_rn(dmb, sdelay[ch]));
    const int a = (sb + shb) & ~3;
    dd_bulk(stage + lane * ROWLEN, in + (size_t)ch * IN_PITCH + a, ROWLEN * 4, bar);
  }
}

#endif  // staging

#if defined(DD_WIN) && DD_WIN
// ============================================================================
// WINDOW mode (host-selected for block_size_x == 32 with strided samples and
// contiguous DMs): a warp's 32 lanes own consecutive samples (lane L:
// s0 + L + 32*i, i < TSX) and ALL share the same TSY consecutive DMs, so
// every shift is warp-uniform.  Adjacent DMs shift by 0 or 1 sample (the
// sweep's slope is < 1 sample per DM), hence for one channel the TSY DMs
// need only the SPAN+1 samples s + sh0 + k (k <= span <= SPAN) per owned
// sample: a lane loads that small window once per channel (coalesced
// 128-byte rows) and reuses every value for all DMs whose offset hits it --
// TSY*TSX adds per TSX*(1+span) loads instead of one load per add.  The
// increment pattern of the TSY shifts (TSY-1 bits) is warp-uniform: one
// indirect branch per channel selects a straight-line block with static
// register offsets.  Patterns (with sh0) are computed 32 channels at a time,
// one channel per lane, and broadcast with a shuffle.  Packed FADD2 adds
// sample pairs; channels are summed in ascending order (bit-exact).
// ============================================================================
#define W (SPAN + 1)
#define NPAT (1 << (TSY - 1))
#define XP ((TSX + 1) / 2)

__host__ __device__ constexpr int dd_popc(int v) { return v ? (v & 1) + dd_popc(v >> 1) : 0; }
// Dense case index of a pattern: patterns ordered by increment count
// (span), then by value -- span 0 is index 0, span 1 are 1..TSY-1, ... --
// so the dispatch can test the frequent small spans first (a switch is
// lowered to a compare tree, never a jump table).  Only spans <= SPAN occur.
__host__ __device__ constexpr int dd_before(int span, int p) {  // patterns < p with this span
  return p == 0 ? 0 : dd_before(span, p - 1) + (dd_popc(p - 1) == span ? 1 : 0);
}
__host__ __device__ constexpr int dd_rank(int p) {
  return dd_before(dd_popc(p), p) + (dd_popc(p) >= 1 ? dd_before(0, NPAT) : 0) +
         (dd_popc(p) >= 2 ? dd_before(1, NPAT) : 0) + (dd_popc(p) >= 3 ? dd_before(2, NPAT) : 0) +
         (dd_popc(p) >= 4 ? dd_before(3, NPAT) : 0) + (dd_popc(p) >= 5 ? dd_before(4, NPAT) : 0) +
         (dd_popc(p) >= 6 ? dd_before(5, NPAT) : 0) + (dd_popc(p) >= 7 ? dd_before(6, NPAT) : 0);
}
__host__ __device__ constexpr int dd_nth(int n, int p = 0) {  // inverse of dd_rank
  return p >= NPAT ? 0 : (dd_rank(p) == n ? p : dd_nth(n, p + 1));
}
// first dense index of each span
#define DD_S1 1
#define DD_S2 (DD_S1 + dd_before(1, NPAT))
#define DD_S3 (DD_S2 + dd_before(2, NPAT))
#define NVALID (DD_S3 + (SPAN >= 3 ? dd_before(3, NPAT) : 0))

struct DdWin {
  float2 acc[TSY][XP];
};

// one channel with increment pattern P (static): load exactly the popc(P)+1
// window samples per owned sample and add them to the TSY DM accumulators
template <int P>
__device__ __forceinline__ void dd_accum(DdWin& st, const float* p) {
  constexpr int span = dd_popc(P);
  float2 x[XP][span + 1];
#pragma unroll
  for (int q = 0; q < XP; ++q)
#pragma unroll
    for (int k = 0; k <= span; ++k) {
      x[q][k].x = p[64 * q + k];
      x[q][k].y = (2 * q + 1 < TSX) ? p[64 * q + 32 + k] : 0.f;
    }
#pragma unroll
  for (int j = 0; j < TSY; ++j) {
    const int g = __popc(P & ((1 << j) - 1));  // offset of DM j (static after unrolling)
#pragma unroll
    for (int q = 0; q < XP; ++q) {
      if (2 * q + 1 < TSX)
        st.acc[j][q] = __fadd2_rn(st.acc[j][q], x[q][g]);
      else
        st.acc[j][q].x = __fadd_rn(st.acc[j][q].x, x[q][g].x);
    }
  }
}

// switch over dense indices LO .. LO+N-1; cases past N have empty bodies and
// fold into `default`, so the compare tree only spans the N live cases
#define DD_CASE(I)                                                 \
  case I:                                                          \
    if constexpr ((I) < N) dd_accum<dd_nth(LO + ((I) < N ? (I) : 0))>(st, p); \
    break;
#define DD_C4(I) DD_CASE(I) DD_CASE(I + 1) DD_CASE(I + 2) DD_CASE(I + 3)
#define DD_C16(I) DD_C4(I) DD_C4(I + 4) DD_C4(I + 8) DD_C4(I + 12)

template <int LO, int N>
__device__ __forceinline__ void dd_switch(DdWin& st, int idx, const float* p) {
  switch (idx - LO) {
    DD_C16(0) DD_C16(16) DD_C16(32) DD_C16(48)
    default:
      break;
  }
}

// frequency-ordered dispatch: span 0 (one pattern, ~1/4 of all channels),
// span 1 (TSY-1 patterns, the most frequent), then spans 2 and 3
__device__ __forceinline__ void dd_dispatch(DdWin& st, int idx, const float* p) {
  if (idx == 0) {
    dd_accum<0>(st, p);
  } else if (SPAN < 2 || idx < DD_S2) {
    dd_switch<DD_S1, (SPAN >= 1 ? DD_S2 - DD_S1 : 0)>(st, idx, p);
  } else if (SPAN < 3 || idx < DD_S3) {
    dd_switch<DD_S2, (SPAN >= 2 ? DD_S3 - DD_S2 : 0)>(st, idx, p);
  } else {
    dd_switch<DD_S3, NVALID - DD_S3>(st, idx, p);
  }
}

// Even tile_size_x: the host splices in a generated inline-PTX dispatch here
// (problems.dd_asm_dispatch: one case per pattern, brx.idx jump table); the
// accumulators are then packed fp32x2 words updated by add.rn.f32x2.
// @DD_ASM_DISPATCH@

extern "C" __global__ void __launch_bounds__(BSX * BSY)
dedispersion_kernel(float* __restrict__ out, const float* __restrict__ in, float dm_first,
                    float dm_step) {
  extern __shared__ __align__(128) float smem[];
  // [stages][CC][ROWLEN] rows | full[NSTAGE] | empty[NSTAGE] | delay[NCH] | pattern->case[NPAT]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + NSTAGE * CC * ROWLEN);
  unsigned long long* empty = bars + NSTAGE;
  float* sdelay = reinterpret_cast<float*>(empty + NSTAGE);
  unsigned char* pidx = reinterpret_cast<unsigned char*>(sdelay + NCH);
  // pattern -> dense case index (span-major, then value): a counting loop
  // (the constexpr dd_rank is recursive -- fine at compile time, a deep
  // call chain at run time)
  for (int p = threadIdx.y * 32 + threadIdx.x; p < NPAT; p += BSX * BSY) {
    const int sp = __popc(p);
    int r = 0;
    for (int q = 0; q < NPAT; ++q) {
      const int sq = __popc(q);
      r += (sq <= SPAN) && (sq < sp || (sq == sp && q < p));
    }
    pidx[p] = (unsigned char)r;
  }
  // per-channel delays in smem: the per-chunk lookups index them by lane
  // (a __constant__ read with 32 different addresses serialises 32-fold)
  for (int c = threadIdx.y * 32 + threadIdx.x; c < NCH; c += BSX * BSY) sdelay[c] = d_delay[c];
  const int lane = threadIdx.x;  // BSX == 32: one warp per DM group
  const int w = threadIdx.y;
  const int sb = (int)blockIdx.y * (32 * TSX);  // block's first sample
  const int db0 = (int)blockIdx.x * (BSY * TSY);  // block's first DM (< NDM)
  const int d0 = db0 + w * TSY;
  const float dmb = __fadd_rn(dm_first, __fmul_rn((float)db0, dm_step));
  if (w == 0 && lane == 0) {
#pragma unroll
    for (int b = 0; b < NSTAGE; ++b) {
      dd_mbar_init(bars + b, 1);       // full: the producer's arrive + TMA bytes
      dd_mbar_init(empty + b, BSY);    // empty: one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nchunks = (NCH + CC - 1) / CC;
  if (w == 0)
    for (int t = 0; t < NSTAGE && t < nchunks; ++t)
      dd_issue_chunk(in, smem + t * CC * ROWLEN, bars + t, t, sb, dmb, lane, sdelay);
#ifdef DD_HAVE_ASM
  unsigned long long acc[TSY][XP];
#pragma unroll
  for (int j = 0; j < TSY; ++j)
#pragma unroll
    for (int q = 0; q < XP; ++q) acc[j][q] = 0ull;  // (+0.0f, +0.0f)
#else
  DdWin st;
#pragma unroll
  for (int j = 0; j < TSY; ++j)
#pragma unroll
    for (int q = 0; q < XP; ++q) st.acc[j][q] = make_float2(0.f, 0.f);
#endif
  for (int t = 0; t < nchunks; ++t) {
    const int stg = t % NSTAGE;
    // lane c: this warp's offset into channel t*CC+c's staged row and the
    // increment pattern of its TSY shifts
    int mine = 0;
    {
      const int ch = t * CC + lane < NCH ? t * CC + lane : NCH - 1;
      const float dl = sdelay[ch];
      // DM values recomputed per chunk (cheaper than 8 live registers);
      // clamped overshoot rows compute a valid DM and are never stored
      const int shb = __float2int_rz(__fmul_rn(dmb, dl));
      const int sh0 = __float2int_rz(__fmul_rn(__fadd_rn(dm_first, __fmul_rn((float)min(d0, NDM - 1), dm_step)), dl));
      int prev = sh0, pat = 0;
#pragma unroll
      for (int j = 1; j < TSY; ++j) {
        const float dmj = __fadd_rn(dm_first, __fmul_rn((float)min(d0 + j, NDM - 1), dm_step));
        const int shj = __float2int_rz(__fmul_rn(dmj, dl));
        pat |= (shj - prev) << (j - 1);  // 0 or 1 (slope < 1 sample per DM)
        prev = shj;
      }
      const int rel = sh0 - shb + ((sb + shb) & 3);  // offset from the aligned row start
      mine = (rel << 8) | pidx[pat];
    }
    dd_mbar_wait(bars + stg, (t / NSTAGE) & 1);
    const float* srow = smem + stg * CC * ROWLEN + lane;
    const int nch = NCH - t * CC < CC ? NCH - t * CC : CC;
#if defined(DD_HAVE_ASM) && !defined(DD_ONE)
    // two channels (in order) per dispatch block: one loop trip and one
    // convergence region per pair (measured: 4.44 -> 4.27 ms at (32,32,4,8,1,0),
    // 6.05 -> 5.82 ms at (32,16,4,8,1,0); a shared-memory slot table instead
    // of the shuffles was slower)
    int c = 0;
#pragma unroll 1
    for (; c + 1 < nch; c += 2, srow += 2 * ROWLEN) {
      const int pk0 = __shfl_sync(0xffffffffu, mine, c);
      const int pk1 = __shfl_sync(0xffffffffu, mine, c + 1);
      dd_asm_dispatch2(acc, pk0 & 0xff, dd_smem_u32(srow + (pk0 >> 8)), pk1 & 0xff,
                       dd_smem_u32(srow + ROWLEN + (pk1 >> 8)));
    }
    if (c < nch) {
      const int pk = __shfl_sync(0xffffffffu, mine, c);
      dd_asm_dispatch(acc, pk & 0xff, dd_smem_u32(srow + (pk >> 8)));
    }
#else
#pragma unroll 1
    for (int c = 0; c < nch; ++c, srow += ROWLEN) {
      const int pk = __shfl_sync(0xffffffffu, mine, c);
#ifdef DD_HAVE_ASM
      dd_asm_dispatch(acc, pk & 0xff, dd_smem_u32(srow + (pk >> 8)));
#else
      dd_dispatch(st, pk & 0xff, srow + (pk >> 8));
#endif
    }
#endif
    // release the stage: one arrival per warp; the producer (warp 0) refills
    // it once all warps have arrived -- the other warps run ahead on the
    // stages already in flight instead of meeting at a block barrier
    __syncwarp();
    if (lane == 0) dd_mbar_arrive(empty + stg);
    if (w == 0 && t + NSTAGE < nchunks) {
      dd_mbar_wait(empty + stg, (t / NSTAGE) & 1);
      dd_issue_chunk(in, smem + stg * CC * ROWLEN, bars + stg, t + NSTAGE, sb, dmb, lane, sdelay);
    }
  }
  const int s0 = sb + lane;
#pragma unroll
  for (int j = 0; j < TSY; ++j) {
    if (d0 + j >= NDM) continue;
    float* o = out + (size_t)(d0 + j) * NSAMP;
#pragma unroll
    for (int q = 0; q < XP; ++q) {
      const int sa = s0 + 64 * q, sbb = sa + 32;
#ifdef DD_HAVE_ASM
      const float2 v = make_float2(__uint_as_float((unsigned)acc[j][q]), __uint_as_float((unsigned)(acc[j][q] >> 32)));
#else
      const float2 v = st.acc[j][q];
#endif
      if (sa < NSAMP) o[sa] = v.x;
      if (2 * q + 1 < TSX && sbb < NSAMP) o[sbb] = v.y;
    }
  }
}

#elif defined(DD_STG) && DD_STG
// ============================================================================
// STAGED generic mode (any block shape; the host selects it when the staged
// rows fit in shared memory): the same per-thread (sample, DM) tiles and
// channel order as the plain generic kernel, but every channel's block-wide
// row segment arrives by TMA bulk copy into a 5-stage ring (as in window
// mode) and the adds read it with LDS: the input stream is prefetched
// instead of each load waiting on L2/HBM (the plain kernel is latency
// bound), and 32 consecutive floats at any alignment are one smem wavefront.
// ============================================================================
extern "C" __global__ void __launch_bounds__(BSX * BSY)
dedispersion_kernel(float* __restrict__ out, const float* __restrict__ in, float dm_first,
                    float dm_step) {
  extern __shared__ __align__(128) float smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + NSTAGE * CC * ROWLEN);
  unsigned long long* empty = bars + NSTAGE;
  float* sdelay = reinterpret_cast<float*>(empty + NSTAGE);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * BSX + tx, lane = tid & 31, w = tid >> 5;
  constexpr int NT = BSX * BSY, NW = (NT + 31) / 32;
  const unsigned wmask = (NT - 32 * w >= 32) ? 0xffffffffu : ((1u << (NT - 32 * w)) - 1u);
  const int sb = (int)blockIdx.y * (BSX * TSX);   // block's first sample
  const int db0 = (int)blockIdx.x * (BSY * TSY);  // block's first DM (< NDM)
  const float dmb = __fadd_rn(dm_first, __fmul_rn((float)db0, dm_step));
  int so[TSX];  // sample offsets within the block
#pragma unroll
  for (int i = 0; i < TSX; ++i) so[i] = STX ? tx + i * BSX : tx * TSX + i;
  int d[TSY];
  float dmv[TSY];
#pragma unroll
  for (int j = 0; j < TSY; ++j) {
    d[j] = db0 + (STY ? ty + j * BSY : ty * TSY + j);
    const int dc = d[j] < NDM ? d[j] : NDM - 1;  // overshoot rows compute a valid DM, never stored
    dmv[j] = __fadd_rn(dm_first, __fmul_rn((float)dc, dm_step));
  }
  for (int c = tid; c < NCH; c += NT) sdelay[c] = d_delay[c];
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < NSTAGE; ++b) {
      dd_mbar_init(bars + b, 1);
      dd_mbar_init(empty + b, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nchunks = (NCH + CC - 1) / CC;
  if (w == 0)
    for (int t = 0; t < NSTAGE && t < nchunks; ++t)
      dd_issue_chunk(in, smem + t * CC * ROWLEN, bars + t, t, sb, dmb, lane, sdelay);
  float acc[TSY][TSX];
#pragma unroll
  for (int j = 0; j < TSY; ++j)
#pragma unroll
    for (int i = 0; i < TSX; ++i) acc[j][i] = 0.f;
  for (int t = 0; t < nchunks; ++t) {
    const int stg = t % NSTAGE;
    dd_mbar_wait(bars + stg, (t / NSTAGE) & 1);
    const float* srow = smem + stg * CC * ROWLEN;
    const int nch = NCH - t * CC < CC ? NCH - t * CC : CC;
#pragma unroll 2
    for (int c = 0; c < nch; ++c, srow += ROWLEN) {
      const float dl = sdelay[t * CC + c];
      const int shb = __float2int_rz(__fmul_rn(dmb, dl));
      const float* row = srow + ((sb + shb) & 3) - shb;  // row[sh + so] = in[ch][sb + so + sh]
#pragma unroll
      for (int j = 0; j < TSY; ++j) {
        const float* p = row + __float2int_rz(__fmul_rn(dmv[j], dl));
#pragma unroll
        for (int i = 0; i < TSX; ++i) acc[j][i] = __fadd_rn(acc[j][i], p[so[i]]);
      }
    }
    __syncwarp(wmask);
    if (lane == 0) dd_mbar_arrive(empty + stg);
    if (w == 0 && t + NSTAGE < nchunks) {
      dd_mbar_wait(empty + stg, (t / NSTAGE) & 1);
      dd_issue_chunk(in, smem + stg * CC * ROWLEN, bars + stg, t + NSTAGE, sb, dmb, lane, sdelay);
    }
  }
#pragma unroll
  for (int j = 0; j < TSY; ++j) {
    if (d[j] >= NDM) continue;
    float* o = out + (size_t)d[j] * NSAMP;
#pragma unroll
    for (int i = 0; i < TSX; ++i)
      if (sb + so[i] < NSAMP) o[sb + so[i]] = acc[j][i];
  }
}

#else  // generic AMBER-style kernel

extern "C" __global__ void __launch_bounds__(BSX * BSY)
dedispersion_kernel(float* __restrict__ out, const float* __restrict__ in, float dm_first,
                    float dm_step) {
  const int tx = threadIdx.x, ty = threadIdx.y;
  int s[TSX];
#pragma unroll
  for (int i = 0; i < TSX; ++i)
    s[i] = (int)blockIdx.y * (BSX * TSX) + (STX ? tx + i * BSX : tx * TSX + i);
  int d[TSY];
  float dmv[TSY];
#pragma unroll
  for (int j = 0; j < TSY; ++j) {
    d[j] = (int)blockIdx.x * (BSY * TSY) + (STY ? ty + j * BSY : ty * TSY + j);
    const int dc = d[j] < NDM ? d[j] : NDM - 1;  // overshoot rows compute a valid DM, never stored
    dmv[j] = __fadd_rn(dm_first, __fmul_rn((float)dc, dm_step));
  }
  float acc[TSY][TSX];
#pragma unroll
  for (int j = 0; j < TSY; ++j)
#pragma unroll
    for (int i = 0; i < TSX; ++i) acc[j][i] = 0.f;

  const float* row = in;
#pragma unroll 2
  for (int ch = 0; ch < NCH; ++ch, row += IN_PITCH) {
    const float dl = d_delay[ch];
#pragma unroll
    for (int j = 0; j < TSY; ++j) {
      const float* p = row + __float2int_rz(__fmul_rn(dmv[j], dl));
#pragma unroll
      for (int i = 0; i < TSX; ++i) acc[j][i] = __fadd_rn(acc[j][i], __ldg(p + s[i]));
    }
  }

#pragma unroll
  for (int j = 0; j < TSY; ++j) {
    if (d[j] >= NDM) continue;
    float* o = out + (size_t)d[j] * NSAMP;
#pragma unroll
    for (int i = 0; i < TSX; ++i)
      if (s[i] < NSAMP) o[s[i]] = acc[j][i];
  }
}

#endif  // DD_WIN

#endif  // REFERENCE_ONLY

// Naive reference: one (dm, sample) per thread; the on-device answer.
extern "C" __global__ void __launch_bounds__(256)
dedispersion_reference(float* __restrict__ out, const float* __restrict__ in, float dm_first,
                       float dm_step) {
  const int s = blockIdx.x * 256 + threadIdx.x;
  const int dm = blockIdx.y;
  if (s >= NSAMP || dm >= NDM) return;
  const float dmv = __fadd_rn(dm_first, __fmul_rn((float)dm, dm_step));
  float acc = 0.f;
  for (int ch = 0; ch < NCH; ++ch)
    acc = __fadd_rn(acc, in[(size_t)ch * IN_PITCH + __float2int_rz(__fmul_rn(dmv, d_delay[ch])) + s]);
  out[(size_t)dm * NSAMP + s] = acc;
}
