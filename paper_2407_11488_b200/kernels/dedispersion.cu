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
