// 2D convolution, tunable (paper Table 1 convolution column;
// space: paper_2407_11488_b200/spaces/convolution.spec, ref
// ts/spaces/convolution.spec:8-23).  NVRTC-compiled per configuration.
//
//   out[y][x] = sum_{i<FH, j<FW} in[y+i][x+j] * filter[i][j]
//
// accumulated as a single fp32 fmaf chain in (i, j) row-major tap order,
// identically in every configuration, in the naive reference kernel
// below and in the CPU oracle (oracle/kernels.c) -- outputs are
// bit-identical across the whole space.
//
// Tunables (compile-time macros):
//   BSX, BSY        thread block
//   TSX, TSY        outputs per thread; a thread owns a CONTIGUOUS
//                   TSX x TSY patch so input rows slide through registers
//                   (each loaded row segment feeds up to TSY output rows)
//   READ_ONLY       global loads through the non-coherent path (ld.global.nc)
//   USE_SHMEM       stage the (TILE+halo) input tile in shared memory
//   USE_PADDING     +1 float per shared row (bank-conflict experiment)
// Problem macros: IMG_W, IMG_H, FW, FH, IN_PITCH (multiple of 4 floats).
// Filter lives in __constant__ d_filter (Kernel Tuner cmem_args).

#ifndef FW
#define FW 15
#endif
#ifndef FH
#define FH 15
#endif

__constant__ float d_filter[FH * FW];

#ifndef REFERENCE_ONLY

#define TILE_W (BSX * TSX)
#define TILE_H (BSY * TSY)
#define SEG (TSX + FW - 1)

// vector width of the per-row segment loads (alignment is provable:
// x origin of every thread is a multiple of TSX, pitches are multiples of 4)
#if USE_PADDING && USE_SHMEM
#define VEC 1
#elif (TSX % 4) == 0
#define VEC 4
#elif (TSX % 2) == 0
#define VEC 2
#else
#define VEC 1
#endif
#define SEG_V (((SEG + VEC - 1) / VEC) * VEC)

#if USE_SHMEM
#define SH_W4 (((TILE_W + FW - 1 + 3) / 4) * 4)
#if USE_PADDING
#define SH_PITCH (SH_W4 + 1)
#else
#define SH_PITCH SH_W4
#endif
#define SH_H (TILE_H + FH - 1)
#endif

template <int V>
__device__ __forceinline__ void load_vec(float* dst, const float* p, bool global_ro);

template <>
__device__ __forceinline__ void load_vec<1>(float* d, const float* p, bool ro) {
  d[0] = ro ? __ldg(p) : *p;
}
template <>
__device__ __forceinline__ void load_vec<2>(float* d, const float* p, bool ro) {
  float2 v = ro ? __ldg(reinterpret_cast<const float2*>(p)) : *reinterpret_cast<const float2*>(p);
  d[0] = v.x;
  d[1] = v.y;
}
template <>
__device__ __forceinline__ void load_vec<4>(float* d, const float* p, bool ro) {
  float4 v = ro ? __ldg(reinterpret_cast<const float4*>(p)) : *reinterpret_cast<const float4*>(p);
  d[0] = v.x;
  d[1] = v.y;
  d[2] = v.z;
  d[3] = v.w;
}

extern "C" __global__ void __launch_bounds__(BSX * BSY)
convolution_kernel(float* __restrict__ out, const float* __restrict__ in) {
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x0 = blockIdx.x * TILE_W;
  const int y0 = blockIdx.y * TILE_H;
  const int ox = x0 + tx * TSX;
  const int oy = y0 + ty * TSY;

#if USE_SHMEM
  extern __shared__ float4 smem4[];
  float* sh = reinterpret_cast<float*>(smem4);
  {
    constexpr int Q = SH_W4 / 4;  // float4 per shared row
    const int tid = ty * BSX + tx;
    for (int i = tid; i < SH_H * Q; i += BSX * BSY) {
      const int r = i / Q;
      const int q = i - r * Q;
      const int gy = y0 + r;
      const int gx = x0 + 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gy < IMG_H + FH - 1 && gx < IN_PITCH) {
        const float4* src = reinterpret_cast<const float4*>(in + (size_t)gy * IN_PITCH + gx);
#if READ_ONLY
        v = __ldg(src);
#else
        v = *src;
#endif
      }
      float* d = sh + r * SH_PITCH + 4 * q;
#if USE_PADDING
      d[0] = v.x;
      d[1] = v.y;
      d[2] = v.z;
      d[3] = v.w;
#else
      *reinterpret_cast<float4*>(d) = v;
#endif
    }
  }
  __syncthreads();
  if (ox >= IMG_W || oy >= IMG_H) return;
  const float* base = sh + (ty * TSY) * SH_PITCH + tx * TSX;
  constexpr int PITCH = SH_PITCH;
  constexpr bool RO = false;
#else
  if (ox >= IMG_W || oy >= IMG_H) return;
  const float* base = in + (size_t)oy * IN_PITCH + ox;
  constexpr int PITCH = IN_PITCH;
  constexpr bool RO = READ_ONLY != 0;
#endif

  float acc[TSY][TSX];
#pragma unroll
  for (int j = 0; j < TSY; ++j)
#pragma unroll
    for (int i = 0; i < TSX; ++i) acc[j][i] = 0.f;

  // input row r of the patch feeds output row j with filter row r-j
#pragma unroll
  for (int r = 0; r < TSY + FH - 1; ++r) {
    float seg[SEG_V];
#pragma unroll
    for (int k = 0; k < SEG_V; k += VEC) load_vec<VEC>(seg + k, base + r * PITCH + k, RO);
#pragma unroll
    for (int j = 0; j < TSY; ++j) {
      const int fi = r - j;
      if (fi >= 0 && fi < FH) {
#pragma unroll
        for (int k = 0; k < FW; ++k) {
          const float f = d_filter[fi * FW + k];
#pragma unroll
          for (int i = 0; i < TSX; ++i) acc[j][i] = fmaf(seg[i + k], f, acc[j][i]);
        }
      }
    }
  }

#pragma unroll
  for (int j = 0; j < TSY; ++j) {
    const int y = oy + j;
    if (y < IMG_H) {
      float* o = out + (size_t)y * IMG_W + ox;
      if (ox + TSX <= IMG_W) {
#if VEC == 4
#pragma unroll
        for (int i = 0; i < TSX; i += 4)
          *reinterpret_cast<float4*>(o + i) = make_float4(acc[j][i], acc[j][i + 1], acc[j][i + 2], acc[j][i + 3]);
#elif VEC == 2
#pragma unroll
        for (int i = 0; i < TSX; i += 2) *reinterpret_cast<float2*>(o + i) = make_float2(acc[j][i], acc[j][i + 1]);
#else
#pragma unroll
        for (int i = 0; i < TSX; ++i) o[i] = acc[j][i];
#endif
      } else {
#pragma unroll
        for (int i = 0; i < TSX; ++i)
          if (ox + i < IMG_W) o[i] = acc[j][i];
      }
    }
  }
}

#endif  // REFERENCE_ONLY

// Naive reference (one output per thread, same fmaf order): produces the
// on-device answer every tuned configuration is verified against.
extern "C" __global__ void __launch_bounds__(256)
convolution_reference(float* __restrict__ out, const float* __restrict__ in) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= IMG_W || y >= IMG_H) return;
  float acc = 0.f;
  for (int i = 0; i < FH; ++i)
    for (int j = 0; j < FW; ++j) acc = fmaf(in[(size_t)(y + i) * IN_PITCH + x + j], d_filter[i * FW + j], acc);
  out[(size_t)y * IMG_W + x] = acc;
}
