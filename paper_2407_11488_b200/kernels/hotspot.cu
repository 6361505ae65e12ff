// Hotspot thermal stencil with temporal tiling (paper Table 1 hotspot
// column; space paper_2407_11488_b200/spaces/hotspot.spec == ref
// ts/spaces/hotspot.spec:11-25).  Rodinia update, clamped (replicate)
// boundary:
//
//   T' = T + sdc * (P + (N + S - 2T) * ry1 + (E + W - 2T) * rx1 + (amb - T) * rz1)
//
// evaluated in exactly this operation order with FMA contraction OFF
// (compiled with --fmad=false) so every configuration, the naive
// reference kernel and the CPU oracle (oracle/kernels.c) agree
// bit-for-bit.  14 FLOP per cell update.
//
// One launch advances the grid by `nsteps` <= TT steps: a block loads
// its (OH+2TT) x (OW+2TT) window (halo TT on each side) into shared
// memory, then ping-pongs between two shared buffers, the valid region
// shrinking by one cell per side per step, and finally writes its
// OH x OW interior.  Tunables:
//   BSX, BSY   thread block
//   TSX, TSY   output cells per thread (OW = BSX*TSX, OH = BSY*TSY)
//   TT         temporal_tiling_factor (steps fused per launch)
//   UNROLL     loop_unroll_factor_t (unroll of the time loop)
//   SH_POWER   stage the power tile in shared memory too
// Work mapping: thread (tx,ty) owns the window columns tx + i*BSX
// (coalesced, conflict-free along x) and a CONTIGUOUS run of RY rows,
// which it sweeps top to bottom keeping N/centre/S in registers, so a
// cell update costs 3 shared loads (S, E, W) instead of 5.
// Problem macros: GW, GH.

#ifndef REFERENCE_ONLY

#define OW (BSX * TSX)
#define OH (BSY * TSY)
#define EW (OW + 2 * TT)
#define EH (OH + 2 * TT)
#define CX ((EW + BSX - 1) / BSX)
#define RY ((EH + BSY - 1) / BSY)

#define STR2(x) #x
#define STR(x) STR2(x)
#define PRAGMA_UNROLL(n) _Pragma(STR(unroll n))

extern "C" __global__ void __launch_bounds__(BSX * BSY)
hotspot_kernel(float* __restrict__ out, const float* __restrict__ tin,
               const float* __restrict__ power, int nsteps, float sdc, float rx1, float ry1,
               float rz1, float amb) {
  extern __shared__ float smem[];
  float* A = smem;
  float* B = smem + EH * EW;
#if SH_POWER
  float* P = smem + 2 * EH * EW;
#endif
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int gx0 = (int)blockIdx.x * OW - TT;
  const int gy0 = (int)blockIdx.y * OH - TT;
  const int r_begin = ty * RY;
  const int r_end = min(r_begin + RY, EH);

  for (int r = r_begin; r < r_end; ++r) {
    const int gy = gy0 + r;
    if (gy < 0 || gy >= GH) continue;
#pragma unroll
    for (int i = 0; i < CX; ++i) {
      const int c = tx + i * BSX;
      const int gx = gx0 + c;
      if (c < EW && gx >= 0 && gx < GW) {
        A[r * EW + c] = __ldg(tin + (size_t)gy * GW + gx);
#if SH_POWER
        P[r * EW + c] = __ldg(power + (size_t)gy * GW + gx);
#endif
      }
    }
  }
  __syncthreads();

PRAGMA_UNROLL(UNROLL)
  for (int s = 0; s < nsteps; ++s) {
    const int lo = s + 1;
    const int hi_r = EH - s - 1;
    const int hi_c = EW - s - 1;
    const int ra = max(r_begin, max(lo, -gy0));          // first active, in-domain row
    const int rb = min(r_end, min(hi_r, GH - gy0));      // one past the last
#pragma unroll
    for (int i = 0; i < CX; ++i) {
      const int c = tx + i * BSX;
      const int gx = gx0 + c;
      if (c < lo || c >= hi_c || gx < 0 || gx >= GW || ra >= rb) continue;
      const bool west_edge = (gx == 0), east_edge = (gx == GW - 1);
      float up = A[(ra - 1) * EW + c];
      float mid = A[ra * EW + c];
      for (int r = ra; r < rb; ++r) {
        const int gy = gy0 + r;
        const float dn = A[(r + 1) * EW + c];
        const float t = mid;
        const float n = (gy == 0) ? t : up;
        const float so = (gy == GH - 1) ? t : dn;
        const float w = west_edge ? t : A[r * EW + c - 1];
        const float e = east_edge ? t : A[r * EW + c + 1];
#if SH_POWER
        const float p = P[r * EW + c];
#else
        const float p = __ldg(power + (size_t)gy * GW + gx);
#endif
        const float c2 = 2.0f * t;
        const float ns = (n + so) - c2;
        const float ew = (e + w) - c2;
        const float z = amb - t;
        float d = p + ns * ry1;
        d = d + ew * rx1;
        d = d + z * rz1;
        B[r * EW + c] = t + sdc * d;
        up = mid;
        mid = dn;
      }
    }
    __syncthreads();
    float* tmp = A;
    A = B;
    B = tmp;
  }

  // write the OH x OW interior (valid after nsteps <= TT steps)
  const int wr0 = max(r_begin, TT), wr1 = min(r_end, TT + OH);
  for (int r = wr0; r < wr1; ++r) {
    const int gy = gy0 + r;
    if (gy >= GH) break;
#pragma unroll
    for (int i = 0; i < CX; ++i) {
      const int c = tx + i * BSX;
      const int gx = gx0 + c;
      if (c >= TT && c < TT + OW && gx < GW) out[(size_t)gy * GW + gx] = A[r * EW + c];
    }
  }
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
  const float c2 = 2.0f * t;
  const float ns = (n + so) - c2;
  const float ew = (e + w) - c2;
  const float z = amb - t;
  float d = power[i] + ns * ry1;
  d = d + ew * rx1;
  d = d + z * rz1;
  out[i] = t + sdc * d;
}
