// Hotspot thermal stencil with temporal tiling (paper Table 1 hotspot
// column; space paper_2407_11488_b200/spaces/hotspot.spec == ref
// ts/spaces/hotspot.spec:11-25), clamped (replicate) boundary.
//
// The naive reference kernel (the on-device answer) computes the Rodinia
// form with explicit fused multiply-adds, 9 FP32 operations per cell:
//
//   T' = fma(sdc, fma(amb-T, rz1, fma(fma(-2,T,E+W), rx1, fma(fma(-2,T,N+S), ry1, P))), T)
//
// The tuned kernels compute the same linear update with the coefficients
// folded on the host (Hotspot.tuned_coefficients, float64 then fp32):
//
//   c  = fma(ap, P, ac)                       ap = sdc, ac = sdc*rz1*amb
//   T' = fma(ax, E+W, fma(ay, N+S, fma(at, T, c)))
//        at = 1 - sdc*(2*rx1 + 2*ry1 + rz1), ay = sdc*ry1, ax = sdc*rx1
//
// -- 5 operations per cell update once c is known; c depends on the power
// row only, so the stream kernels compute it once per row and launch (the
// first level that reads a power row replaces it by c in the shared ring)
// and the block-tile kernels once per cell and launch.  Every tuned
// configuration uses this operation order, and so does the CPU oracle's
// oracle_hotspot_tuned (oracle/kernels.c), compiled without implicit
// contraction (--fmad=false): tuned results agree with it bit-for-bit, and
// with the Rodinia chain within the north_star tolerance (rtol 1e-5;
// measured 1.4e-6 norm-wise at 1024^2 x 20 steps).
//
// One launch advances the grid by `nsteps` <= TT steps: a block owns an
// OH x OW output tile plus a halo of TT cells per side (window EH x EW),
// stages it on chip, advances it nsteps times -- the valid region
// shrinking by one cell per side per step -- and writes the interior.
//
// Tunables: BSX, BSY (block), TSX, TSY (cells per thread: OW = BSX*TSX,
// OH = BSY*TSY), TT (temporal_tiling_factor), UNROLL
// (loop_unroll_factor_t, unroll of the time loop), SH_POWER (stage the
// power tile in shared memory; else re-read it through L1 each step).
//
// Thread (tx, ty) owns window columns tx + i*BSX (coalesced, bank-
// conflict free) and a CONTIGUOUS run of RY rows.  Two schedules,
// chosen at compile time from the register budget:
//   REGISTER mode (small per-thread footprint): the thread owns PAIRS of
//     adjacent columns held in float2 registers across all steps; N/S come
//     from its own registers, only E/W (and the strip ends) are exchanged
//     through a ping-pong pair of shared buffers; arithmetic is packed
//     FFMA2/FADD2 (sm_100): per 2 cells 2 LDS + 1 STS.64 + 9 packed ops,
//     1 barrier per step; sh_power keeps the power tile in registers.
//   SHARED mode (large tiles): cells live in the shared ping-pong pair;
//     rows are swept top-down, each row updating the thread's CX columns
//     (independent -> ILP) with per-column N/C/S windows in registers:
//     3 LDS + 1 STS per cell update.
// Blocks whose window lies fully inside the grid take a branch-free
// path; only edge blocks evaluate the clamping selects.
// Problem macros: GW, GH.

#define HS_STEP(t, n, s, e, w, p, sdc, rx1, ry1, rz1, amb)                              \
  fmaf((sdc),                                                                            \
       fmaf((amb) - (t), (rz1),                                                          \
            fmaf(fmaf(-2.0f, (t), (e) + (w)), (rx1), fmaf(fmaf(-2.0f, (t), (n) + (s)), (ry1), (p)))), \
       (t))

// tuned form (see the header): power term, then the 5-operation update
#define HS_C(p, ap, ac) fmaf((ap), (p), (ac))
#define HS_FAST(t, n, s, e, w, c, at, ay, ax) fmaf((ax), (e) + (w), fmaf((ay), (n) + (s), fmaf((at), (t), (c))))

#ifndef REFERENCE_ONLY

struct HsCoef {
  float at, ay, ax, ap, ac;
};

#if defined(HS_STREAM) && HS_STREAM
// ============================================================================
// STREAM mode (the host selects it when the register/smem budget allows).
//
// The unit of work is a WARP, not a block: warp w streams down a strip of
// SW = 32*TSX window columns (lane L owns the TSX contiguous columns
// L*TSX..L*TSX+TSX-1) and produces the UW useful columns of a segment of
// `segh` output rows.  The host sizes segments from the kernel's measured
// occupancy so the grid is TSY whole waves (TSY = 1: one wave, the
// tallest segments, least vertical halo).  The nsteps <= TT time levels are pipelined along the stream
// (time skewing): when input row i arrives, level k is advanced at row
// i-k for k = 1..nsteps, so every level keeps only a 3-row ring in
// registers (R[k][3][.]) and level nsteps leaves the pipeline one row per
// iteration.  Neighbours: N/S from the register ring, E/W of the lane's
// edge columns by warp shuffles (2 SHFL per lane per level): no block
// barrier and no shared-memory exchange.  Halo cost: the strip recomputes
// TA+TT columns (UW = floor4(SW - TA - TT) useful) and each segment streams
// segh + 2*nsteps rows.
//
// Memory: every lane stages ITS OWN columns, so no lane ever waits for
// another: input rows arrive by cp.async (LDGSTS, 16/8/4-byte chunks,
// zero-fill outside the grid) into an NR-row per-warp shared ring, NR-1
// rows in flight, completion by per-thread cp.async groups (no mbarrier,
// no __syncwarp).  SH_POWER=1 stages power rows the same way in a PR-row
// ring (each power row serves TT levels); SH_POWER=0 re-reads power
// through L1 per level.  Output rows leave by direct vector stores (window
// origin and UW are multiples of 4 columns, so every 16-byte chunk is
// aligned and either fully useful or not).  Chunks are laid out
// chunk-major in shared memory (bank-conflict-free vector LDS).
// Arithmetic is packed FFMA2/FADD2 on column pairs, per component
// identical to HS_FAST (bit-exact).
//
// loop_unroll_factor_t: the level loop is always fully unrolled (its
// registers are indexed by level); UNROLL == 1 streams one row per
// iteration (3-slot register rings, 3 ring phases), UNROLL > 1 two rows
// per iteration (two independent chains per level, 4-slot rings, 2 phases).  Mapping of the tunables: block = (BSX, BSY) threads = WPB warps
// taking consecutive warp tiles (strip-fastest), TSX = columns per lane,
// TSY = waves of warp tiles (row segments per strip = TSY x the count that
// fills one wave), TT = levels per launch.
// ============================================================================

#define SW (32 * TSX)
#define TA (((TT) + 3) & ~3)
#define UW (((SW - TA - TT) / 4) * 4)
#define NSTRIPS ((GW + UW - 1) / UW)
// Stream kernels are compiled per THREAD COUNT, not per (BSX, BSY): the
// unit of work is a warp, so block shape and TSY (waves, a launch-geometry
// choice) never reach the code -- configurations that differ only there
// share one cubin (problems.Hotspot.config_defines).  The thread count
// stays a compile-time launch bound: ptxas schedules differently under
// __launch_bounds__(64) and (256) even though both cap at 255 registers
// (measured: 680 vs 781 instructions in the interior loop), so blocks of
// different sizes must not share code.
#define NTHREADS (HS_THREADS)
// input ring: NR rows = NG groups of 2 rows (one group per iteration),
// NG-1 groups in flight
#ifndef HS_NR
#define HS_NR 8
#endif
#define NR HS_NR
#define NG (NR / 2)
// power rows are prefetched PD rows ahead of their first use (level 1),
// independently of the input ring depth: the power ring must hold rows from
// the deepest level's (i - TT) to the newest staged one, so a shallower
// power prefetch shrinks it (TT=8, NR=16: 32 -> 16 rows at PD=6) and raises
// the warps resident per SM.  Default PD = NR - 2 (power staged with input).
#ifndef HS_PD
#define HS_PD (NR - 2)
#endif
#define PD HS_PD
// power ring: a power of two >= TT + PD + 2 rows, preceded by TT-1 MIRROR
// rows: row r lives in slot (r - ia + 1) & (PR - 1) -- the two power rows an
// iteration first reads (i-1, i) never straddle the wrap -- and the first
// level to read a row writes its power term c into the slot and, for the
// last TT-1 slots, also into the mirror row slot - PR (in front of slot 0).
// Every later level then reads row i-k at ONE per-iteration base pointer
// minus a compile-time offset, never wrapping (no per-level slot arithmetic).
#define PM (SH_POWER ? (TT - 1) : 0)
#define PR (SH_POWER ? ((TT + PD + 2) <= 8 ? 8 : ((TT + PD + 2) <= 16 ? 16 : ((TT + PD + 2) <= 32 ? 32 : 64))) : 0)
// HS_STREAM == 2 ("smem rings"): the level rings live in per-warp shared
// memory instead of registers (configurations whose TT x TSX register rings
// exceed the __launch_bounds__ budget); one row per iteration
#if HS_STREAM == 2
#define LR (TT * 3)
#else
#define LR 0
#endif
#define WARP_FLOATS (SW * (NR + PM + PR + LR))
// staging chunk (floats) and chunks per lane
#define CW ((TSX % 4) == 0 ? 4 : ((TSX % 2) == 0 ? 2 : 1))
#define NCH (TSX / CW)
#define NP2 ((TSX + 1) / 2)
// rows per stream iteration: loop_unroll_factor_t > 1 unrolls the row stream
// by two (two independent update chains per level)
#if HS_STREAM == 2
#define HS_RPI 1
#else
#define HS_RPI ((UNROLL) > 1 ? 2 : 1)
#endif
#define COL(v, j) ((j) % 2 == 0 ? (v)[(j) / 2].x : (v)[(j) / 2].y)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// one staging chunk, zero-filled when `bytes` == 0 (outside the grid)
__device__ __forceinline__ void cp_chunk(float* dst, const float* src, unsigned bytes) {
#if CW == 4
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
#elif CW == 2
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
#else
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
#endif
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct HsK2 {
  float2 at, ay, ax, ap, ac;
};

__device__ __forceinline__ HsK2 hs_pairs(const HsCoef& k) {
  return HsK2{make_float2(k.at, k.at), make_float2(k.ay, k.ay), make_float2(k.ax, k.ax), make_float2(k.ap, k.ap),
              make_float2(k.ac, k.ac)};
}

struct HsStream {
  const float* tin;
  const float* power;
  float* out;
  float* tring;   // NR rows, chunk-major
  float* pring;   // PR rows (SH_POWER)
  float* lring;   // HS_STREAM == 2: level rings [TT][3] rows, chunk-major
  int lane, gx0, ia, ib, y0, y1, nsteps;
  unsigned nst;      // rows ia .. ia+nst are staged (ia+nst = min(ib, GH-1))
  int cbytes[NCH];   // staging bytes per chunk (0 outside the grid)
  int csrc[NCH];     // global column of each chunk (clamped into the grid)
  unsigned omask;    // chunks that are useful output columns
  unsigned lmask, rmask;  // owned cells at gx == 0 / gx == GW-1
  bool xl, xr;            // this lane's first / last column is grid column 0 / GW-1
};

// chunk c of this lane inside a shared row (chunk-major: lanes contiguous)
__device__ __forceinline__ float* chunk_ptr(float* row, int c, int lane) { return row + (c * 32 + lane) * CW; }

__device__ __forceinline__ void lds_pairs(float2 (&v)[NP2], const float* row, int lane) {
  float t[TSX];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const float* p = row + (c * 32 + lane) * CW;
#if CW == 4
    const float4 q = *reinterpret_cast<const float4*>(p);
    t[4 * c] = q.x; t[4 * c + 1] = q.y; t[4 * c + 2] = q.z; t[4 * c + 3] = q.w;
#elif CW == 2
    const float2 q = *reinterpret_cast<const float2*>(p);
    t[2 * c] = q.x; t[2 * c + 1] = q.y;
#else
    t[c] = *p;
#endif
  }
#pragma unroll
  for (int q = 0; q < NP2; ++q) v[q] = make_float2(t[2 * q], 2 * q + 1 < TSX ? t[2 * q + 1] : 0.f);
}

// inverse of lds_pairs: this lane's columns into a chunk-major shared row
__device__ __forceinline__ void sts_pairs(float* row, const float2 (&v)[NP2], int lane) {
  float t[TSX];
#pragma unroll
  for (int j = 0; j < TSX; ++j) t[j] = COL(v, j);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    float* p = row + (c * 32 + lane) * CW;
#if CW == 4
    *reinterpret_cast<float4*>(p) = make_float4(t[4 * c], t[4 * c + 1], t[4 * c + 2], t[4 * c + 3]);
#elif CW == 2
    *reinterpret_cast<float2*>(p) = make_float2(t[2 * c], t[2 * c + 1]);
#else
    *p = t[c];
#endif
  }
}

// stage input row `row` into the input ring (no commit)
__device__ __forceinline__ void hs_stage_t(const HsStream& S, int row) {
  if ((unsigned)(row - S.ia) <= S.nst) {  // ia <= row <= min(ib, GH-1): one compare
    const size_t rb = (size_t)row * GW;
    float* tr = S.tring + ((row - S.ia) & (NR - 1)) * SW;
#pragma unroll
    for (int c = 0; c < NCH; ++c) cp_chunk(chunk_ptr(tr, c, S.lane), S.tin + rb + S.csrc[c], S.cbytes[c]);
  }
}

// stage power row `row` into the power ring (no commit); rows before the
// stream start are never read as valid data (garbage pipeline rows)
__device__ __forceinline__ void hs_stage_p(const HsStream& S, int row) {
#if SH_POWER
  if ((unsigned)(row - S.ia) <= S.nst) {
    const size_t rb = (size_t)row * GW;
    float* pr = S.pring + ((row - S.ia + 1) & (PR - 1)) * SW;
#pragma unroll
    for (int c = 0; c < NCH; ++c) cp_chunk(chunk_ptr(pr, c, S.lane), S.power + rb + S.csrc[c], S.cbytes[c]);
  }
#else
  (void)S;
  (void)row;
#endif
}

// The staging group of stream iteration i (one cp.async group per
// iteration, always committed so the group count stays uniform):
//   two rows per iteration: input rows i+NR-2, i+NR-1, power rows i+PD-1,
//   i+PD; iteration i first reads power rows i-1, i (staged PD/2 groups
//   earlier) and input rows i, i+1 (NG-1 groups earlier; PD <= NR-2).
//   one row per iteration: input row i+NR-1, power row i+PD-1; iteration i
//   first reads power row i-1 (PD groups earlier) and input row i.
__device__ __forceinline__ void hs_stage_iter2(const HsStream& S, int i) {
  // (one slot computation and row address per ring and pair instead of per
  // row saved 3% of the T=7 loop's instructions but measured 15% slower at
  // T=5 -- profiles/round2/hs_ring/hs_exp_t5.jsonl; kept per row)
  hs_stage_t(S, i + NR - 2);
  hs_stage_t(S, i + NR - 1);
  hs_stage_p(S, i + PD - 1);
  hs_stage_p(S, i + PD);
  cp_commit();
}
__device__ __forceinline__ void hs_stage_iter1(const HsStream& S, int i) {
  hs_stage_t(S, i + NR - 1);
  hs_stage_p(S, i + PD - 1);
  cp_commit();
}
static_assert(PD >= 0 && PD <= NR - 2, "power prefetch must not outrun the input ring");
static_assert(HS_RPI == 1 || PD % 2 == 0, "two rows per iteration: even power prefetch distance");
static_assert(!SH_POWER || PR >= TT + PD + 2, "power ring too small");
#define HS_WAIT2 ((PD) / 2)
#define HS_WAIT1 (PD)

// The power term c = fma(ap, P, ac) of row r for this lane's columns.
// SH_POWER: the first level to read a power row (FRESH) turns the staged P
// into c in place -- the lane's own columns of the ring, so no other lane
// is involved -- and the later levels read c.  Without SH_POWER every level
// re-reads P through L1 and forms c itself.
template <bool FRESH>
__device__ __forceinline__ void hs_power(float2 (&pw)[NP2], const HsStream& S, float* prow, int r,
                                         bool mirror, const HsK2& k2) {
#if SH_POWER
  (void)r;
  lds_pairs(pw, prow, S.lane);
  if (FRESH) {
#pragma unroll
    for (int q = 0; q < NP2; ++q) pw[q] = __ffma2_rn(k2.ap, pw[q], k2.ac);
    sts_pairs(prow, pw, S.lane);                      // the slot ...
    if (mirror) sts_pairs(prow - PR * SW, pw, S.lane);  // ... and its mirror (warp-uniform)
  }
#else
  (void)prow;
  (void)mirror;
  const float* grow = S.power + (size_t)min(max(r, 0), GH - 1) * GW;
  float t[TSX];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const float* p = grow + S.csrc[c];
#if CW == 4
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    t[4 * c] = q.x; t[4 * c + 1] = q.y; t[4 * c + 2] = q.z; t[4 * c + 3] = q.w;
#elif CW == 2
    const float2 q = __ldg(reinterpret_cast<const float2*>(p));
    t[2 * c] = q.x; t[2 * c + 1] = q.y;
#else
    t[c] = __ldg(p);
#endif
  }
#pragma unroll
  for (int q = 0; q < NP2; ++q)
    pw[q] = __ffma2_rn(k2.ap, make_float2(t[2 * q], 2 * q + 1 < TSX ? t[2 * q + 1] : 0.f), k2.ac);
#endif
}

// this iteration's power slot ps (of row i-1) and base pointer; row i-k
// (k >= 1) of an earlier level is at pbase - (k - 1) * SW (slot or mirror)
__device__ __forceinline__ int hs_pslot(const HsStream& S, int i) { return SH_POWER ? ((i - S.ia) & (PR - 1)) : 0; }
#define HS_PROW(pb, k) ((pb) - (SH_POWER ? ((k) - 1) * SW : 0))
#define HS_MIRRORED(slot) ((slot) > PR - TT)

// One cell-pair row update (HS_FAST on columns 2q, 2q+1; bit-exact):
// C = centre row, N/S rows, wl/er = W of column 0 / E of column TSX-1
// (from the neighbour lanes), P = the row's power term c.
// Edge modes E (warp-uniform, chosen per warp tile):
//   E & 3 == 0: interior strip (no horizontal clamp)
//   E & 3 == 1: strip holding grid column 0 / GW-1 at a LANE boundary: the
//               clamp is applied once per level to the shuffled neighbour
//               value (wl/er), not per cell
//   E & 3 == 2: boundary inside a lane's columns: per-cell selects
//   E & 4     : top/bottom row segment: N/S clamps at rows 0 / GH-1
template <int E>
__device__ __forceinline__ void hs_row_update(float2 (&nv)[NP2], const float2* N, const float2* Cc,
                                              const float2* Sr, float wl, float er, const float2 (&P)[NP2],
                                              bool top, bool bot, const HsStream& S, const HsCoef& kk,
                                              const HsK2& k2) {
#pragma unroll
  for (int q = 0; q < NP2; ++q) {
    const int j = 2 * q;
    const float2 t = Cc[q];
    float2 n = N[q], s = Sr[q];
    // west / east neighbours of columns j and j+1 straddle the register
    // pairs: form them as scalars and add them with two scalar FADDs (the
    // FMA-pipe cost of one FADD2) instead of moving registers into pairs
    float w0 = (j == 0) ? wl : COL(Cc, j - 1);
    float e0 = (j + 1 < TSX) ? t.y : er;
    float w1 = t.x;
    float e1 = (j + 2 < TSX) ? COL(Cc, j + 2) : er;
    if (E & 4) {
      n = top ? t : n;
      s = bot ? t : s;
    }
    if ((E & 3) == 2) {
      w0 = (S.lmask >> j) & 1u ? t.x : w0;
      e0 = (S.rmask >> j) & 1u ? t.x : e0;
      w1 = (S.lmask >> (j + 1)) & 1u ? t.y : w1;
      e1 = (S.rmask >> (j + 1)) & 1u ? t.y : e1;
    }
    if (j + 1 < TSX) {
      const float2 ns = __fadd2_rn(n, s);
      const float2 ew = make_float2(__fadd_rn(e0, w0), __fadd_rn(e1, w1));
      float2 u = __ffma2_rn(k2.at, t, P[q]);
      u = __ffma2_rn(k2.ay, ns, u);
      nv[q] = __ffma2_rn(k2.ax, ew, u);
    } else {  // odd TSX: scalar last column
      nv[q] = make_float2(HS_FAST(t.x, n.x, s.x, e0, w0, P[q].x, kk.at, kk.ay, kk.ax), 0.f);
    }
  }
}

__device__ __forceinline__ void hs_store_row(const HsStream& S, int ro, const float2 (&cur)[NP2]) {
  if (ro >= S.y0 && ro < S.y1) {
    float v[TSX];
#pragma unroll
    for (int j = 0; j < TSX; ++j) v[j] = COL(cur, j);
    float* orow = S.out + (size_t)ro * GW;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if ((S.omask >> c) & 1u) {
        float* p = orow + S.csrc[c];
#if CW == 4
        *reinterpret_cast<float4*>(p) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
#elif CW == 2
        *reinterpret_cast<float2*>(p) = make_float2(v[2 * c], v[2 * c + 1]);
#else
        *p = v[c];
#endif
      }
    }
  }
}

// One stream iteration: input rows i, i+1 arrive; level k advances rows
// a = i-k and b = i+1-k (two independent chains per level).  Level k-1
// rows a-1, a live in the 4-slot register ring; rows a+1, a+2 are the
// two fresh rows the previous level just produced (they then replace the
// dead slots of rows a-3, a-2).  Slots: row x at (x - ia) & 3, static for
// PH = ((i - ia) / 2) & 1.
template <int PH, int E, int NS>
__device__ __forceinline__ void hs_stream_iter(const HsStream& S, float2 (&R)[TT][4][NP2], int i,
                                               const HsCoef& kk, const HsK2& k2) {
  hs_stage_iter2(S, i);  // keep NG-1 input row pairs in flight
  cp_wait<HS_WAIT2>();   // this lane's chunks of input rows i, i+1 and power rows i-1, i have landed
  float2 f0[NP2], f1[NP2];       // fresh rows of the previous level (level 0: input)
  const float* tb = S.tring + ((i - S.ia) & (NR - 1)) * SW;  // rows i, i+1 (even slot: no wrap)
  const int ps = hs_pslot(S, i);
  float* pbase = S.pring + ps * SW;
  lds_pairs(f0, tb, S.lane);  // rows >= GH: stale, never used
  lds_pairs(f1, tb + SW, S.lane);
  // E/W neighbours of every level's OLD centre row (level k-1 row a),
  // hoisted into one convergence block
  float wla[TT], era[TT];
  float2 pprev[NP2];  // power row of the previous level's row a
#pragma unroll
  for (int k = 1; k <= TT; ++k) {
    const int sC = ((2 * PH - k) % 4 + 4) % 4;
    wla[k - 1] = __shfl_up_sync(0xffffffffu, COL(R[k - 1][sC], TSX - 1), 1);
    era[k - 1] = __shfl_down_sync(0xffffffffu, R[k - 1][sC][0].x, 1);
    if ((E & 3) == 1) {  // grid column 0 / GW-1 sits at this lane's edge: clamp = own value
      wla[k - 1] = S.xl ? R[k - 1][sC][0].x : wla[k - 1];
      era[k - 1] = S.xr ? COL(R[k - 1][sC], TSX - 1) : era[k - 1];
    }
  }
#pragma unroll
  for (int k = 1; k <= TT; ++k) {
    if (k > NS) break;  // static level count: no exit phis
    const int a = i - k;
    const int sN = ((2 * PH - k - 1) % 4 + 4) % 4;  // row a-1
    const int sC = ((2 * PH - k) % 4 + 4) % 4;      // row a
    const int s0 = ((2 * PH - k + 1) % 4 + 4) % 4;  // row a+1 (fresh f0)
    const int s1 = ((2 * PH - k + 2) % 4 + 4) % 4;  // row a+2 (fresh f1)
    // E/W of the fresh centre row a+1 (row b's centre)
    float wlb = __shfl_up_sync(0xffffffffu, COL(f0, TSX - 1), 1);
    float erb = __shfl_down_sync(0xffffffffu, f0[0].x, 1);
    if ((E & 3) == 1) {
      wlb = S.xl ? f0[0].x : wlb;
      erb = S.xr ? COL(f0, TSX - 1) : erb;
    }
    // power rows a and a+1; row a+1 is the previous level's row a (reuse)
    float2 pa[NP2], pb[NP2];
    if (k == 1) {  // rows a, a+1 are new to the pipeline: P -> c
      hs_power<true>(pa, S, pbase, a, HS_MIRRORED(ps), k2);
      hs_power<true>(pb, S, pbase + SW, a + 1, HS_MIRRORED(ps + 1), k2);
    } else {
      hs_power<false>(pa, S, HS_PROW(pbase, k), a, false, k2);
#pragma unroll
      for (int q = 0; q < NP2; ++q) pb[q] = pprev[q];
    }
#pragma unroll
    for (int q = 0; q < NP2; ++q) pprev[q] = pa[q];
    float2 na[NP2], nb[NP2];
    hs_row_update<E>(na, R[k - 1][sN], R[k - 1][sC], f0, wla[k - 1], era[k - 1], pa, (E & 4) && a == 0,
                        (E & 4) && a == GH - 1, S, kk, k2);
    hs_row_update<E>(nb, R[k - 1][sC], f0, f1, wlb, erb, pb, (E & 4) && a + 1 == 0, (E & 4) && a + 1 == GH - 1, S,
                        kk, k2);
#pragma unroll
    for (int q = 0; q < NP2; ++q) {
      R[k - 1][s0][q] = f0[q];
      R[k - 1][s1][q] = f1[q];
      f0[q] = na[q];
      f1[q] = nb[q];
    }
  }
  // f0, f1 = level nsteps at rows i - nsteps, i + 1 - nsteps
  const int ro = i - NS;
  hs_store_row(S, ro, f0);
  hs_store_row(S, ro + 1, f1);
}

// ---- smem level rings (HS_STREAM == 2) --------------------------------------
// Same pipeline as hs_stream_iter1, but level k-1's rows a-1, a are read
// from a 3-row ring in this warp's shared memory and the fresh row (in
// registers) is written back to it.  Each lane only ever touches its own
// columns there (E/W still come from shuffles), so no warp sync is needed.
#if HS_STREAM == 2
template <int PH, int E, int NS>
__device__ __forceinline__ void hs_stream_iter_s(const HsStream& S, int i, const HsCoef& kk, const HsK2& k2) {
  hs_stage_iter1(S, i);
  cp_wait<HS_WAIT1>();
  float2 f0[NP2];
  const int ps = hs_pslot(S, i);
  float* pbase = S.pring + ps * SW;
  lds_pairs(f0, S.tring + ((i - S.ia) & (NR - 1)) * SW, S.lane);  // rows >= GH: stale, never used
#pragma unroll
  for (int k = 1; k <= TT; ++k) {
    if (k > NS) break;
    const int a = i - k;
    const int sN = ((PH - k - 1) % 3 + 3) % 3;
    const int sC = ((PH - k) % 3 + 3) % 3;
    const int s0 = ((PH - k + 1) % 3 + 3) % 3;
    float* ring = S.lring + (k - 1) * 3 * SW;
    sts_pairs(ring + s0 * SW, f0, S.lane);  // level k-1 row a+1
    float2 N[NP2], Cc[NP2];
    lds_pairs(N, ring + sN * SW, S.lane);
    lds_pairs(Cc, ring + sC * SW, S.lane);
    float wl = __shfl_up_sync(0xffffffffu, COL(Cc, TSX - 1), 1);
    float er = __shfl_down_sync(0xffffffffu, Cc[0].x, 1);
    if ((E & 3) == 1) {
      wl = S.xl ? Cc[0].x : wl;
      er = S.xr ? COL(Cc, TSX - 1) : er;
    }
    float2 pa[NP2];
    if (k == 1)
      hs_power<true>(pa, S, pbase, a, HS_MIRRORED(ps), k2);
    else
      hs_power<false>(pa, S, HS_PROW(pbase, k), a, false, k2);
    float2 na[NP2];
    hs_row_update<E>(na, N, Cc, f0, wl, er, pa, (E & 4) && a == 0, (E & 4) && a == GH - 1, S, kk, k2);
#pragma unroll
    for (int q = 0; q < NP2; ++q) f0[q] = na[q];
  }
  hs_store_row(S, i - NS, f0);
}

template <int E, int NS>
__device__ __forceinline__ void hs_stream_run_s(const HsStream& S, const HsCoef& kk) {
  const HsK2 k2 = hs_pairs(kk);
  for (int i = S.ia; i <= S.ib; i += 3) {
    hs_stream_iter_s<0, E, NS>(S, i, kk, k2);
    if (i + 1 > S.ib) break;
    hs_stream_iter_s<1, E, NS>(S, i + 1, kk, k2);
    if (i + 2 > S.ib) break;
    hs_stream_iter_s<2, E, NS>(S, i + 2, kk, k2);
  }
}
#endif

// ---- one row per iteration (loop_unroll_factor_t == 1) --------------------
// Level k-1 keeps rows a-1, a in a 3-slot ring (row x at (x - ia) mod 3,
// static for PH = (i - ia) mod 3); the fresh row a+1 arrives from level k-1.
template <int PH, int E, int NS>
__device__ __forceinline__ void hs_stream_iter1(const HsStream& S, float2 (&R)[TT][3][NP2], int i,
                                                const HsCoef& kk, const HsK2& k2) {
  hs_stage_iter1(S, i);  // keep NR-1 input rows in flight (one group per row)
  cp_wait<HS_WAIT1>();
  float2 f0[NP2];
  const int ps = hs_pslot(S, i);
  float* pbase = S.pring + ps * SW;
  lds_pairs(f0, S.tring + ((i - S.ia) & (NR - 1)) * SW, S.lane);  // rows >= GH: stale, never used
  float wla[TT], era[TT];  // E/W of every level's centre row, one convergence block
#pragma unroll
  for (int k = 1; k <= TT; ++k) {
    const int sC = ((PH - k) % 3 + 3) % 3;
    wla[k - 1] = __shfl_up_sync(0xffffffffu, COL(R[k - 1][sC], TSX - 1), 1);
    era[k - 1] = __shfl_down_sync(0xffffffffu, R[k - 1][sC][0].x, 1);
    if ((E & 3) == 1) {  // grid column 0 / GW-1 sits at this lane's edge: clamp = own value
      wla[k - 1] = S.xl ? R[k - 1][sC][0].x : wla[k - 1];
      era[k - 1] = S.xr ? COL(R[k - 1][sC], TSX - 1) : era[k - 1];
    }
  }
#pragma unroll
  for (int k = 1; k <= TT; ++k) {
    if (k > NS) break;
    const int a = i - k;
    const int sN = ((PH - k - 1) % 3 + 3) % 3;
    const int sC = ((PH - k) % 3 + 3) % 3;
    const int s0 = ((PH - k + 1) % 3 + 3) % 3;
    float2 pa[NP2];
    if (k == 1)
      hs_power<true>(pa, S, pbase, a, HS_MIRRORED(ps), k2);
    else
      hs_power<false>(pa, S, HS_PROW(pbase, k), a, false, k2);
    float2 na[NP2];
    hs_row_update<E>(na, R[k - 1][sN], R[k - 1][sC], f0, wla[k - 1], era[k - 1], pa, (E & 4) && a == 0,
                        (E & 4) && a == GH - 1, S, kk, k2);
#pragma unroll
    for (int q = 0; q < NP2; ++q) {
      R[k - 1][s0][q] = f0[q];
      f0[q] = na[q];
    }
  }
  hs_store_row(S, i - NS, f0);
}

template <int E, int NS>
__device__ __forceinline__ void hs_stream_run1(const HsStream& S, const HsCoef& kk) {
  const HsK2 k2 = hs_pairs(kk);
  float2 R[TT][3][NP2];
#pragma unroll
  for (int a = 0; a < TT; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int q = 0; q < NP2; ++q) R[a][b][q] = make_float2(0.f, 0.f);
  for (int i = S.ia; i <= S.ib; i += 3) {
    hs_stream_iter1<0, E, NS>(S, R, i, kk, k2);
    if (i + 1 > S.ib) break;
    hs_stream_iter1<1, E, NS>(S, R, i + 1, kk, k2);
    if (i + 2 > S.ib) break;
    hs_stream_iter1<2, E, NS>(S, R, i + 2, kk, k2);
  }
}

// ---- two rows per iteration (loop_unroll_factor_t > 1) -----------------------
#ifndef HS_P4
#define HS_P4 ((TT) <= 7)
#endif
template <int E, int NS>
__device__ __forceinline__ void hs_stream_run(const HsStream& S, const HsCoef& kk) {
  const HsK2 k2 = hs_pairs(kk);
  float2 R[TT][4][NP2];
#pragma unroll
  for (int a = 0; a < TT; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < NP2; ++q) R[a][b][q] = make_float2(0.f, 0.f);
#if HS_P4
  // four iterations per loop trip (two ring periods) for the interior
  // tiles: ptxas coalesces the loop-carried rings instead of emitting ~45
  // register moves at every back edge (interior loop 626 -> 577 SASS per 4
  // rows at T=7; measured T=7 0.1474 -> 0.1420 ms).  Only for TT <= 7: at
  // TT = 10 the longer body spills (0.150 -> 0.199 ms), at TT = 8 it is even.
  // Full-depth launches only (NS == TT): the single remainder launch keeps
  // the shorter loop -- one stream-loop copy less for NVRTC per configuration
  if (E == 0 && NS == TT) {
    for (int i = S.ia; i <= S.ib; i += 8) {
      hs_stream_iter<0, E, NS>(S, R, i, kk, k2);
      if (i + 2 > S.ib) break;
      hs_stream_iter<1, E, NS>(S, R, i + 2, kk, k2);
      if (i + 4 > S.ib) break;
      hs_stream_iter<0, E, NS>(S, R, i + 4, kk, k2);
      if (i + 6 > S.ib) break;
      hs_stream_iter<1, E, NS>(S, R, i + 6, kk, k2);
    }
    return;
  }
#endif
  for (int i = S.ia; i <= S.ib; i += 4) {
    hs_stream_iter<0, E, NS>(S, R, i, kk, k2);
    if (i + 2 > S.ib) break;
    hs_stream_iter<1, E, NS>(S, R, i + 2, kk, k2);
  }
}

// One launch advancing NS (static) levels.  The full-depth launches of a run
// use hotspot_kernel (NS = TT); the remainder launch of ceil(20/TT) uses
// hotspot_rem_kernel (NS = HS_REM), so no code path has a runtime level
// count -- a dynamic-depth path needs ~1.6x the registers (exit phis) and,
// being part of the same kernel, would cap every launch's occupancy.
//
// Warp tiles.  Strips whose window touches a grid border (a prefix
// [0, XL) and a suffix [XR, NSTRIPS), from the compile-time geometry) run
// the all-selects edge code, ~1.6x the interior's instructions per row, so
// the host gives them proportionally more, shorter row segments (nse per
// edge strip vs ns per interior strip) and all warps of the single wave
// finish together.  Edge-strip tiles take the first warp indices.
#define XL ((TA) / (UW) + 1 < NSTRIPS ? (TA) / (UW) + 1 : NSTRIPS)
#define XR_RAW ((GW - 1 - SW + TA) < 0 ? 0 : (GW - 1 - SW + TA) / (UW) + 1)
#define XR (XR_RAW < XL ? XL : (XR_RAW > NSTRIPS ? NSTRIPS : XR_RAW))
#define NXE (XL + NSTRIPS - XR)
#define NXI (XR - XL)
template <int NS>
__device__ __forceinline__ void hs_stream_body(float* __restrict__ out, const float* __restrict__ tin,
                                               const float* __restrict__ power, float at, float ay,
                                               float ax, float ap, float ac, int segh, int nsegs,
                                               int segh0, int seghe, int nsegse, int segh0e) {
  extern __shared__ __align__(128) float smem[];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int wid = tid >> 5;
  const int g = (int)blockIdx.x * (int)((blockDim.x * blockDim.y) >> 5) + wid;
  int strip, seg;
  if (g < NXE * nsegse) {  // edge strips
    const int e = g % NXE;
    strip = e < XL ? e : XR + (e - XL);
    seg = g / NXE;
    segh = seghe;
    nsegs = nsegse;
    segh0 = segh0e;
  } else {
    const int h = g - NXE * nsegse;
    if (NXI == 0 || h >= NXI * nsegs) return;  // whole warp; no block barrier follows
    strip = XL + h % NXI;
    seg = h / NXI;
  }
  HsStream S;
  S.lane = tid & 31;
  S.tin = tin;
  S.power = power;
  S.out = out;
  S.tring = smem + wid * WARP_FLOATS;
  S.pring = S.tring + (NR + PM) * SW;  // slot 0, after the mirror rows
  S.lring = S.pring + PR * SW;
  S.gx0 = strip * UW - TA;
  S.nsteps = NS;
  // segments: the first (and, by the host's choice of segh, the last) are
  // shorter -- their warps pay the N/S boundary selects, so all warps of the
  // single wave finish together
  S.y0 = seg == 0 ? 0 : segh0 + (seg - 1) * segh;
  S.y1 = seg == nsegs - 1 ? GH : min(S.y0 + (seg == 0 ? segh0 : segh), GH);
  S.ia = max(0, S.y0 - NS);
  S.ib = S.y1 - 1 + NS;
  S.nst = (unsigned)(min(S.ib, GH - 1) - S.ia);
  S.omask = S.lmask = S.rmask = 0u;
  S.xl = S.gx0 + S.lane * TSX == 0;
  S.xr = S.gx0 + S.lane * TSX + TSX - 1 == GW - 1;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int wc = S.lane * TSX + c * CW;  // window column of the chunk
    const int gx = S.gx0 + wc;
    const bool in = gx >= 0 && gx < GW;   // chunks never straddle the grid edge (GW % 4 == 0)
    S.cbytes[c] = in ? 4 * CW : 0;
    S.csrc[c] = in ? gx : 0;
    if (wc >= TA && wc < TA + UW && gx < GW) S.omask |= 1u << c;
  }
#pragma unroll
  for (int j = 0; j < TSX; ++j) {
    const int gx = S.gx0 + S.lane * TSX + j;
    if (gx == 0) S.lmask |= 1u << j;
    if (gx == GW - 1) S.rmask |= 1u << j;
  }
  // programmatic dependent launch: wait until the previous launch of the
  // run -- the producer of `tin` and reader of `out` -- has completed and
  // its writes are visible (a no-op without the launch attribute, i.e. for
  // the first launch of a run).  Everything above overlaps its drain.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // prologue: the staging groups of the virtual iterations before ia
#if HS_RPI == 2
  for (int g2 = 0; g2 < NG - 1; ++g2) hs_stage_iter2(S, S.ia - (NR - 2) + 2 * g2);
#else
  for (int j = S.ia - (NR - 1); j < S.ia; ++j) hs_stage_iter1(S, j);
#endif
  const HsCoef kk{at, ay, ax, ap, ac};
  // edge mode of this warp tile (see hs_row_update)
  const bool xedge = S.gx0 <= 0 || S.gx0 + SW > GW - 1;
  const bool yedge = S.ia == 0 || S.ib >= GH - 1;
#if HS_STREAM == 2
#define HS_RUN hs_stream_run_s
#elif HS_RPI == 2
#define HS_RUN hs_stream_run
#else
#define HS_RUN hs_stream_run1
#endif
  // two instantiated edge modes per kernel (each one is a full copy of the
  // stream loop, and NVRTC time grows with every copy: 7 -> 4 copies per
  // configuration halved the compile time): interior, and the all-selects
  // code for every tile touching a border -- edge strips get shorter
  // segments (above), top/bottom segments are short (STREAM_EDGE_SEG)
  if (!xedge && !yedge)
    HS_RUN<0, NS>(S, kk);
  else
    HS_RUN<6, NS>(S, kk);
  cp_wait<0>();  // no copy may land in smem after the warp has left
  // let the next launch be scheduled once every warp has finished its stream
  // (triggering at the start instead placed the next grid's CTAs early and
  // measured 1-4% slower than this; no trigger at all: 1-4% slower too --
  // profiles/round2/hs_ring/hs_exp_pdl2.jsonl)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

extern "C" __global__ void __launch_bounds__(NTHREADS)
hotspot_kernel(float* __restrict__ out, const float* __restrict__ tin,
               const float* __restrict__ power, int nsteps, float at, float ay, float ax,
               float ap, float ac, int segh, int nsegs, int segh0, int seghe, int nsegse, int segh0e) {
  (void)nsteps;  // == TT
  hs_stream_body<TT>(out, tin, power, at, ay, ax, ap, ac, segh, nsegs, segh0, seghe, nsegse, segh0e);
}

#if defined(HS_REM) && HS_REM > 0
extern "C" __global__ void __launch_bounds__(NTHREADS)
hotspot_rem_kernel(float* __restrict__ out, const float* __restrict__ tin,
                   const float* __restrict__ power, int nsteps, float at, float ay, float ax,
                   float ap, float ac, int segh, int nsegs, int segh0, int seghe, int nsegse,
                   int segh0e) {
  (void)nsteps;  // == HS_REM
  hs_stream_body<HS_REM>(out, tin, power, at, ay, ax, ap, ac, segh, nsegs, segh0, seghe, nsegse, segh0e);
}
#endif

#else  // !HS_STREAM

#define OW (BSX * TSX)
#define OH (BSY * TSY)
#define EW (OW + 2 * TT)
#define EH (OH + 2 * TT)
#define CX ((EW + BSX - 1) / BSX)
#define RY ((EH + BSY - 1) / BSY)
#define NTHREADS (BSX * BSY)

#define STR2(x) #x
#define STR(x) STR2(x)
#define PRAGMA_UNROLL(n) _Pragma(STR(unroll n))

// register budget per thread under __launch_bounds__(NTHREADS)
#define REG_BUDGET ((65536 / NTHREADS) > 255 ? 255 : (65536 / NTHREADS))
// register mode works on PAIRS of adjacent columns (float2, packed FFMA2):
// CXP pairs per thread, 2 (value) + 2 (new value) + 2*SH_POWER (power)
// registers per pair
#define CXP ((EW + 2 * BSX - 1) / (2 * BSX))
#define REG_PAIRS_MAX (((REG_BUDGET - 40) / (4 + 2 * SH_POWER)) < 16 ? ((REG_BUDGET - 40) / (4 + 2 * SH_POWER)) : 16)
// padded window: row pitch SP floats, thread-row strips of RY rows SS
// floats apart; SS = RY*SP + a skew so that the 32/BSX thread rows sharing
// a warp hit disjoint bank groups with 8-byte accesses (SS = 2*BSX*odd
// (mod 4*BSX) when 2*BSX < 32) -- no bank conflicts
#define SP (2 * CXP * BSX)
#define RT (RY * BSY)
#define PSKEW_M (4 * BSX)
#define SKEW ((2 * BSX >= 32) ? 0 : ((2 * BSX - ((RY * SP) % PSKEW_M) + PSKEW_M) % PSKEW_M))
#define SS (RY * SP + SKEW)
#define REG_GUARD (SP + 34)
#define REG_SMEM_BYTES (4 * (2 * BSY * SS + 3 * REG_GUARD))
// (mirrored on the host by problems.Hotspot.kernel_mode / smem_bytes)
#define SKEW_M (2 * BSX)
#if !defined(HS_FORCE_SHARED) && (CXP * RY <= REG_PAIRS_MAX) && (REG_SMEM_BYTES <= 200 * 1024)
#define HS_REGISTER_MODE 1
#define HS_BUF (BSY * SS)
#define HS_GUARD REG_GUARD
#else
#define HS_REGISTER_MODE 0
// shared mode: row r lives at ROWB(r); thread-row strips of RY rows are
// SSS floats apart, SSS = RY*EW + a skew making the 32/BSX strips that
// share a warp hit disjoint bank groups (same rule as register mode)
#define SKEW_S ((BSX >= 32) ? 0 : ((BSX - ((RY * EW) % SKEW_M) + SKEW_M) % SKEW_M))
#define SSS (RY * EW + SKEW_S)
#define ROWB(r) (((r) / RY) * SSS + ((r) % RY) * EW)
#define HS_BUF (BSY * SSS)
#define HS_GUARD (EW + 1)
#endif

#if HS_REGISTER_MODE

// Register mode: thread (tx,ty) owns column PAIRS (2p, 2p+1), p = tx + i*BSX,
// over a contiguous strip of RY rows, values held in float2 registers across
// all steps.  A step per pair: 2 scalar LDS (W of the left column, E of the
// right one; N/S come from registers except at strip ends), the 5
// arithmetic ops of HS_FAST as PACKED fp32x2 instructions (FFMA2/FADD2,
// sm_100; per component identical to the scalar fmaf/fadd -> bit-exact),
// and one 8-byte STS.  Rows with no active cell in the warp are skipped
// (warp-uniform vote).  Smem is a padded, skewed layout (no bank
// conflicts) with guard bands absorbing the border over-reach.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

struct HsCoef2 {  // coefficient pairs, built once per launch
  float2 at, ay, ax, ap, ac;
};

// HS_FAST on a column pair; c = the cells' power term
__device__ __forceinline__ float2 hs_step2(float2 t, float2 n, float2 s, float2 e, float2 w, float2 c,
                                           const HsCoef2& k) {
  float2 u = __ffma2_rn(k.at, t, c);
  u = __ffma2_rn(k.ay, __fadd2_rn(n, s), u);
  return __ffma2_rn(k.ax, __fadd2_rn(e, w), u);
}

template <bool EDGE>
__device__ __forceinline__ void hs_reg_steps(float2 (&v)[CXP][RY], const float2 (&pw)[CXP][RY],
                                             const float* __restrict__ power, float* A, float* B,
                                             int nsteps, int tx, int ty, int gx0, int gy0, HsCoef kk) {
  const HsCoef2 k{f2(kk.at, kk.at), f2(kk.ay, kk.ay), f2(kk.ax, kk.ax), f2(kk.ap, kk.ap), f2(kk.ac, kk.ac)};
  const int tb = ty * SS + 2 * tx;
  const int r0 = ty * RY;
  PRAGMA_UNROLL(UNROLL)
  for (int s = 0; s < nsteps; ++s) {
    const int lo = s + 1;
    float2 nv[CXP][RY];
    bool ok0[CXP], ok1[CXP];
#pragma unroll
    for (int i = 0; i < CXP; ++i) {
      const int c0 = 2 * (tx + i * BSX);
      ok0[i] = (c0 >= lo) && (c0 < EW - lo);
      ok1[i] = (c0 + 1 >= lo) && (c0 + 1 < EW - lo);
      if (EDGE) {
        ok0[i] = ok0[i] && (gx0 + c0 >= 0) && (gx0 + c0 < GW);
        ok1[i] = ok1[i] && (gx0 + c0 + 1 >= 0) && (gx0 + c0 + 1 < GW);
      }
    }
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const int r = r0 + j;
      bool row_ok = (r >= lo) && (r < EH - lo);
      if (EDGE) row_ok = row_ok && (gy0 + r >= 0) && (gy0 + r < GH);
      if (__any_sync(0xffffffffu, row_ok)) {
        const float* aj = A + tb + j * SP;
        float* bj = B + tb + j * SP;
#pragma unroll
        for (int i = 0; i < CXP; ++i) {
          const float2 t = v[i][j];
          float2 n = (j > 0) ? v[i][j - 1]
                             : *reinterpret_cast<const float2*>(aj + 2 * i * BSX + (RY - 1) * SP - SS);
          float2 so = (j < RY - 1) ? v[i][j + 1]
                                   : *reinterpret_cast<const float2*>(aj + 2 * i * BSX + SS - (RY - 1) * SP);
          float2 w = f2(aj[2 * i * BSX - 1], t.x);
          float2 e = f2(t.y, aj[2 * i * BSX + 2]);
          float2 p;
          if (EDGE) {
            const int gx = gx0 + 2 * (tx + i * BSX), gy = gy0 + r;
            n = (gy == 0) ? t : n;
            so = (gy == GH - 1) ? t : so;
            w.x = (gx == 0) ? t.x : w.x;
            w.y = (gx + 1 == 0) ? t.y : w.y;
            e.x = (gx == GW - 1) ? t.x : e.x;
            e.y = (gx + 1 == GW - 1) ? t.y : e.y;
          }
#if SH_POWER
          p = pw[i][j];
#else
          {
            int gyp = gy0 + r, gxp = gx0 + 2 * (tx + i * BSX);
            int gxq = gxp + 1;
            if (EDGE) {
              gyp = min(max(gyp, 0), GH - 1);
              gxp = min(max(gxp, 0), GW - 1);
              gxq = min(max(gxq, 0), GW - 1);
            }
            p = f2(HS_C(__ldg(power + (size_t)gyp * GW + gxp), kk.ap, kk.ac),
                   HS_C(__ldg(power + (size_t)gyp * GW + gxq), kk.ap, kk.ac));
          }
#endif
          const float2 u = hs_step2(t, n, so, e, w, p, k);
          nv[i][j] = f2((row_ok && ok0[i]) ? u.x : t.x, (row_ok && ok1[i]) ? u.y : t.y);
          *reinterpret_cast<float2*>(bj + 2 * i * BSX) = nv[i][j];
        }
      } else {
        // no active cell of this row in the warp: unchanged, and never read
        // by an active cell of a later step (the active region only shrinks)
#pragma unroll
        for (int i = 0; i < CXP; ++i) nv[i][j] = v[i][j];
      }
    }
#pragma unroll
    for (int i = 0; i < CXP; ++i)
#pragma unroll
      for (int j = 0; j < RY; ++j) v[i][j] = nv[i][j];
    __syncthreads();
    float* tmp = A;
    A = B;
    B = tmp;
  }
}

#else  // SHARED mode

// Rows outer, the thread's CX columns inner: every row iteration updates
// CX independent cells (ILP), each column keeping its N/C/S sliding window
// in registers (3 LDS + 1 STS per update).  Columns outside the active
// region read a clamped (valid) column and skip the store.
template <bool EDGE>
__device__ __forceinline__ float* hs_smem_steps(const float* __restrict__ power, float* A, float* B,
                                                const float* P, int nsteps, int tx, int r_begin,
                                                int r_end, int gx0, int gy0, HsCoef k) {
  int cl[CX];
#pragma unroll
  for (int i = 0; i < CX; ++i) cl[i] = min(tx + i * BSX, EW - 1);
  PRAGMA_UNROLL(UNROLL)
  for (int s = 0; s < nsteps; ++s) {
    const int lo = s + 1;
    int ra = max(r_begin, lo), rb = min(r_end, EH - lo);
    if (EDGE) {
      ra = max(ra, -gy0);
      rb = min(rb, GH - gy0);
    }
    bool cok[CX];
    float up[CX], mid[CX];
    const int rl = min(ra, EH - 1);  // padding threads (ra >= rb) must still read in bounds
#pragma unroll
    for (int i = 0; i < CX; ++i) {
      const int c = tx + i * BSX;
      cok[i] = (c >= lo) && (c < EW - lo);
      if (EDGE) cok[i] = cok[i] && (gx0 + c >= 0) && (gx0 + c < GW);
      up[i] = A[ROWB(rl - 1) + cl[i]];
      mid[i] = A[ROWB(rl) + cl[i]];
    }
#pragma unroll 2
    for (int r = ra; r < rb; ++r) {
      const int rowb = ROWB(r);
      const float* ar = A + rowb;
      const float* an = A + ROWB(r + 1);
#pragma unroll
      for (int i = 0; i < CX; ++i) {
        const int c = cl[i];
        const float dn = an[c];
        const float t = mid[i];
        float n = up[i], so = dn, w = ar[c - 1], e = ar[c + 1];
        if (EDGE) {
          const int gy = gy0 + r, gx = gx0 + c;
          n = (gy == 0) ? t : n;
          so = (gy == GH - 1) ? t : so;
          w = (gx == 0) ? t : w;
          e = (gx == GW - 1) ? t : e;
        }
#if SH_POWER
        const float p = P[rowb + c];  // staged as c
#else
        int gxp = gx0 + c;
        if (EDGE) gxp = min(max(gxp, 0), GW - 1);
        const float p = HS_C(__ldg(power + (size_t)(gy0 + r) * GW + gxp), k.ap, k.ac);
#endif
        const float u = HS_FAST(t, n, so, e, w, p, k.at, k.ay, k.ax);
        if (cok[i]) B[rowb + c] = u;
        up[i] = t;
        mid[i] = dn;
      }
    }
    __syncthreads();
    float* tmp = A;
    A = B;
    B = tmp;
  }
  return A;
}

#endif

extern "C" __global__ void __launch_bounds__(NTHREADS)
hotspot_kernel(float* __restrict__ out, const float* __restrict__ tin,
               const float* __restrict__ power, int nsteps, float at, float ay, float ax,
               float ap, float ac) {
  extern __shared__ float smem[];
  // [guard][A][guard][B][guard][P], each buffer HS_BUF floats; the guards
  // absorb register mode's one-row/one-column overreach at the borders
  float* A = smem + HS_GUARD;
  float* B = A + HS_BUF + HS_GUARD;
  float* P = B + HS_BUF + HS_GUARD;  // shared mode with SH_POWER only
  (void)P;
  const HsCoef k{at, ay, ax, ap, ac};
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int gx0 = (int)blockIdx.x * OW - TT;
  const int gy0 = (int)blockIdx.y * OH - TT;
  const int r_begin = ty * RY;
  const int r_end = min(r_begin + RY, EH);

#if HS_REGISTER_MODE
  // interior: the whole PADDED window maps inside the grid (padding cells
  // then read valid global addresses and need no clamping)
  const bool interior = gx0 >= 0 && gy0 >= 0 && gx0 + SP <= GW && gy0 + RT <= GH;
  float2 v[CXP][RY];
  float2 pw[CXP][RY];
  const int tb = ty * SS + 2 * tx;
#pragma unroll
  for (int i = 0; i < CXP; ++i) {
    const int gx = gx0 + 2 * (tx + i * BSX);
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const int gy = gy0 + r_begin + j;
      const bool in_y = interior || (gy >= 0 && gy < GH);
      const bool in0 = in_y && (interior || (gx >= 0 && gx < GW));
      const bool in1 = in_y && (interior || (gx + 1 >= 0 && gx + 1 < GW));
      const size_t o = (size_t)gy * GW + gx;
      v[i][j] = f2(in0 ? __ldg(tin + o) : 0.f, in1 ? __ldg(tin + o + 1) : 0.f);
#if SH_POWER
      pw[i][j] = f2(HS_C(in0 ? __ldg(power + o) : 0.f, ap, ac), HS_C(in1 ? __ldg(power + o + 1) : 0.f, ap, ac));
#else
      pw[i][j] = f2(0.f, 0.f);
#endif
      *reinterpret_cast<float2*>(A + tb + j * SP + 2 * i * BSX) = v[i][j];
    }
  }
  __syncthreads();
  if (interior)
    hs_reg_steps<false>(v, pw, power, A, B, nsteps, tx, ty, gx0, gy0, k);
  else
    hs_reg_steps<true>(v, pw, power, A, B, nsteps, tx, ty, gx0, gy0, k);
#pragma unroll
  for (int i = 0; i < CXP; ++i) {
    const int c = 2 * (tx + i * BSX);
    const int gx = gx0 + c;
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const int r = r_begin + j;
      const int gy = gy0 + r;
      if (r >= TT && r < TT + OH && gy < GH) {
        if (c >= TT && c < TT + OW && gx < GW) out[(size_t)gy * GW + gx] = v[i][j].x;
        if (c + 1 >= TT && c + 1 < TT + OW && gx + 1 < GW) out[(size_t)gy * GW + gx + 1] = v[i][j].y;
      }
    }
  }
#else
  for (int r = r_begin; r < r_end; ++r) {
    const int gy = gy0 + r;
    if (gy < 0 || gy >= GH) continue;
#pragma unroll
    for (int i = 0; i < CX; ++i) {
      const int c = tx + i * BSX;
      const int gx = gx0 + c;
      if (c < EW && gx >= 0 && gx < GW) {
        A[ROWB(r) + c] = __ldg(tin + (size_t)gy * GW + gx);
#if SH_POWER
        P[ROWB(r) + c] = HS_C(__ldg(power + (size_t)gy * GW + gx), ap, ac);
#endif
      }
    }
  }
  __syncthreads();
  const bool edge = gx0 < 0 || gy0 < 0 || gx0 + EW > GW || gy0 + EH > GH;
  float* R = edge ? hs_smem_steps<true>(power, A, B, P, nsteps, tx, r_begin, r_end, gx0, gy0, k)
                  : hs_smem_steps<false>(power, A, B, P, nsteps, tx, r_begin, r_end, gx0, gy0, k);
  const int wr0 = max(r_begin, TT), wr1 = min(r_end, TT + OH);
  for (int r = wr0; r < wr1; ++r) {
    const int gy = gy0 + r;
    if (gy >= GH) break;
#pragma unroll
    for (int i = 0; i < CX; ++i) {
      const int c = tx + i * BSX;
      const int gx = gx0 + c;
      if (c >= TT && c < TT + OW && gx < GW) out[(size_t)gy * GW + gx] = R[ROWB(r) + c];
    }
  }
#endif
}

#endif  // HS_STREAM

#endif  // REFERENCE_ONLY

// Naive reference: one step per launch, one cell per thread, global
// memory only; the on-device answer for verification.
extern "C" __global__ void __launch_bounds__(256)
hotspot_reference(float* __restrict__ out, const float* __restrict__ tin,
                  const float* __restrict__ power, float sdc, float rx1, float ry1, float rz1,
                  float amb) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= GW || y >= GH) return;
  const size_t i = (size_t)y * GW + x;
  const float t = tin[i];
  const float n = y > 0 ? tin[i - GW] : t;
  const float so = y < GH - 1 ? tin[i + GW] : t;
  const float w = x > 0 ? tin[i - 1] : t;
  const float e = x < GW - 1 ? tin[i + 1] : t;
  out[i] = HS_STEP(t, n, so, e, w, power[i], sdc, rx1, ry1, rz1, amb);
}
