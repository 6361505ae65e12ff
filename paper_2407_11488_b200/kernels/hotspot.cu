// Hotspot thermal stencil with temporal tiling (paper Table 1 hotspot
// column; space paper_2407_11488_b200/spaces/hotspot.spec == ref
// ts/spaces/hotspot.spec:11-25).  Rodinia update, clamped (replicate)
// boundary, written with explicit fused multiply-adds:
//
//   T' = fma(sdc, fma(amb-T, rz1, fma(fma(-2,T,E+W), rx1, fma(fma(-2,T,N+S), ry1, P))), T)
//
// (15 FLOP per cell update).  The same operation order is used by every
// configuration, by the naive reference kernel and by the CPU oracle
// (oracle/kernels.c), compiled without implicit contraction
// (--fmad=false), so results agree bit-for-bit.
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
//   REGISTER mode (CX*RY small): the thread's cells live in registers
//     across all steps; N/S neighbours come from its own registers, only
//     E/W (and the strip ends) are exchanged through a ping-pong pair of
//     shared buffers: 2 LDS + 1 STS per cell update, 1 barrier per step.
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

#ifndef REFERENCE_ONLY

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
#define REG_CELLS_MAX (((REG_BUDGET - 40) / 2) < 32 ? ((REG_BUDGET - 40) / 2) : 32)
// padded window of register mode: row pitch SP, RT rows; each thread-row
// strip of RY rows starts SS floats after the previous one, SS = RY*SP +
// a skew chosen so that the 32/BSX thread rows sharing a warp land on
// disjoint bank groups (SS = BSX * odd (mod 32)) -- no bank conflicts.
#define SP (CX * BSX)
#define RT (RY * BSY)
#define SKEW_M (2 * BSX)
#define SKEW ((BSX >= 32) ? 0 : ((BSX - ((RY * SP) % SKEW_M) + SKEW_M) % SKEW_M))
#define SS (RY * SP + SKEW)
#define REG_GUARD (SP + 33)
#define REG_SMEM_BYTES (4 * ((2 + SH_POWER) * BSY * SS + 3 * REG_GUARD))
// (mirrored on the host by problems.Hotspot.kernel_mode / smem_bytes)
#if !defined(HS_FORCE_SHARED) && (CX * RY <= REG_CELLS_MAX) && (REG_SMEM_BYTES <= 200 * 1024)
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

struct HsCoef {
  float sdc, rx1, ry1, rz1, amb;
};

#if HS_REGISTER_MODE

// Register mode works on a PADDED window: row pitch SP = CX*BSX and RT =
// RY*BSY rows, so every thread cell (i, j) has its own smem slot at the
// affine index tb + j*SP + i*BSX (compile-time offsets from one per-thread
// base).  Cells are computed branch-free; activity (the shrinking valid
// region, domain edges) is one select per cell from per-row / per-column
// predicates evaluated once per step, and rows with no active cell in the
// warp are skipped with a warp-uniform test.  Guard bands of SP+1 floats
// before/after each buffer keep the +-1 / +-SP reads of border cells in
// bounds; those values only ever feed inactive (discarded) cells.
template <bool EDGE>
__device__ __forceinline__ void hs_reg_steps(float (&v)[CX][RY], const float* __restrict__ power,
                                             float* A, float* B, const float* P, int nsteps,
                                             int tx, int r0, int gx0, int gy0, HsCoef k) {
  const int tb = (r0 / RY) * SS + tx;  // strip of thread row r0/RY
  PRAGMA_UNROLL(UNROLL)
  for (int s = 0; s < nsteps; ++s) {
    const int lo = s + 1;
    float nv[CX][RY];
    bool col_ok[CX];
#pragma unroll
    for (int i = 0; i < CX; ++i) {
      const int c = tx + i * BSX;
      col_ok[i] = (c >= lo) && (c < EW - lo);
      if (EDGE) col_ok[i] = col_ok[i] && (gx0 + c >= 0) && (gx0 + c < GW);
    }
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const int r = r0 + j;
      bool row_ok = (r >= lo) && (r < EH - lo);
      if (EDGE) row_ok = row_ok && (gy0 + r >= 0) && (gy0 + r < GH);
      float* bj = B + tb + j * SP;
      if (__any_sync(0xffffffffu, row_ok)) {
        const float* aj = A + tb + j * SP;
#pragma unroll
        for (int i = 0; i < CX; ++i) {
          const float t = v[i][j];
          // strip ends: the neighbour row lives in the adjacent strip
          float n = (j > 0) ? v[i][j - 1] : aj[i * BSX + (RY - 1) * SP - SS];
          float so = (j < RY - 1) ? v[i][j + 1] : aj[i * BSX + SS - (RY - 1) * SP];
          float w = aj[i * BSX - 1];
          float e = aj[i * BSX + 1];
          if (EDGE) {
            const int gx = gx0 + tx + i * BSX, gy = gy0 + r;
            n = (gy == 0) ? t : n;
            so = (gy == GH - 1) ? t : so;
            w = (gx == 0) ? t : w;
            e = (gx == GW - 1) ? t : e;
          }
#if SH_POWER
          const float p = P[tb + j * SP + i * BSX];
#else
          int gyp = gy0 + r, gxp = gx0 + tx + i * BSX;
          if (EDGE) {
            gyp = min(max(gyp, 0), GH - 1);
            gxp = min(max(gxp, 0), GW - 1);
          }
          const float p = __ldg(power + (size_t)gyp * GW + gxp);
#endif
          const float u = HS_STEP(t, n, so, e, w, p, k.sdc, k.rx1, k.ry1, k.rz1, k.amb);
          nv[i][j] = (row_ok && col_ok[i]) ? u : t;
          bj[i * BSX] = nv[i][j];
        }
      } else {
#pragma unroll
        for (int i = 0; i < CX; ++i) {
          nv[i][j] = v[i][j];
          bj[i * BSX] = v[i][j];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CX; ++i)
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
        const float p = P[rowb + c];
#else
        int gxp = gx0 + c;
        if (EDGE) gxp = min(max(gxp, 0), GW - 1);
        const float p = __ldg(power + (size_t)(gy0 + r) * GW + gxp);
#endif
        const float u = HS_STEP(t, n, so, e, w, p, k.sdc, k.rx1, k.ry1, k.rz1, k.amb);
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
               const float* __restrict__ power, int nsteps, float sdc, float rx1, float ry1,
               float rz1, float amb) {
  extern __shared__ float smem[];
  // [guard][A][guard][B][guard][P], each buffer HS_BUF floats; the guards
  // absorb register mode's one-row/one-column overreach at the borders
  float* A = smem + HS_GUARD;
  float* B = A + HS_BUF + HS_GUARD;
  float* P = B + HS_BUF + HS_GUARD;  // used only when SH_POWER
  const HsCoef k{sdc, rx1, ry1, rz1, amb};
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int gx0 = (int)blockIdx.x * OW - TT;
  const int gy0 = (int)blockIdx.y * OH - TT;
  const int r_begin = ty * RY;
  const int r_end = min(r_begin + RY, EH);

#if HS_REGISTER_MODE
  // interior: the whole PADDED window maps inside the grid (padding cells
  // then read valid global addresses and need no clamping)
  const bool interior = gx0 >= 0 && gy0 >= 0 && gx0 + SP <= GW && gy0 + RT <= GH;
  float v[CX][RY];
  const int tb = ty * SS + tx;
#pragma unroll
  for (int i = 0; i < CX; ++i) {
    const int c = tx + i * BSX;
    const int gx = gx0 + c;
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const int gy = gy0 + r_begin + j;
      v[i][j] = 0.f;
      if (interior || (gx >= 0 && gx < GW && gy >= 0 && gy < GH)) {
        v[i][j] = __ldg(tin + (size_t)gy * GW + gx);
#if SH_POWER
        P[tb + j * SP + i * BSX] = __ldg(power + (size_t)gy * GW + gx);
#endif
      }
      A[tb + j * SP + i * BSX] = v[i][j];
    }
  }
  __syncthreads();
  if (interior)
    hs_reg_steps<false>(v, power, A, B, P, nsteps, tx, r_begin, gx0, gy0, k);
  else
    hs_reg_steps<true>(v, power, A, B, P, nsteps, tx, r_begin, gx0, gy0, k);
#pragma unroll
  for (int i = 0; i < CX; ++i) {
    const int c = tx + i * BSX;
    const int gx = gx0 + c;
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const int r = r_begin + j;
      const int gy = gy0 + r;
      if (c >= TT && c < TT + OW && r >= TT && r < TT + OH && gx < GW && gy < GH)
        out[(size_t)gy * GW + gx] = v[i][j];
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
        P[ROWB(r) + c] = __ldg(power + (size_t)gy * GW + gx);
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
