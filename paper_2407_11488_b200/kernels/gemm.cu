// Single-precision GEMM, CLBlast xgemm parameterisation (paper Table 2;
// space paper_2407_11488_b200/spaces/gemm.spec == ref
// ts/spaces/gemm.spec:8-32), SIMT FFMA on sm_100a.
//
// Storage (BLAS column-major with A transposed, the layout CLBlast's
// kernel consumes, so vector loads run along M for A/C and N for B):
//   a(m,k) = A[k*GM + m]    b(k,n) = B[k*GN + n]    c(m,n) = C[n*GM + m]
//   c(m,n) = sum_k a(m,k) * b(k,n)
// Every configuration accumulates each c(m,n) as ONE fmaf chain over
// k = 0..K-1 in order, so all configurations, the reference kernel and
// the CPU oracle are bit-identical.
//
// Tunables (CLBlast names):
//   MWG, NWG, KWG    block tile (M, N, K)
//   MDIMC, NDIMC     compute threads: block = MDIMC*NDIMC threads,
//                    each owning MWI x NWI = (MWG/MDIMC) x (NWG/NDIMC) outputs
//   MDIMA, NDIMB     thread re-shape for the cooperative A / B tile loads
//   VWM, VWN         vector widths along M (A loads, C stores) / N (B)
//   STRM, STRN       1: a thread's vectors are strided by MDIMC*VWM
//                    (NDIMC*VWN) -- coalesced; 0: contiguous per thread
//   SA, SB           stage the A / B k-tile in shared memory (else read
//                    global memory directly inside the k loop); staged
//                    tiles are double-buffered (dynamic smem) with a
//                    register prefetch of the next k-tile
// Problem macros: GM, GN, GK.

#ifndef REFERENCE_ONLY

#define MWI (MWG / MDIMC)
#define MP ((MWI + 1) / 2)
#define NWI (NWG / NDIMC)
#define KDIMA ((MDIMC * NDIMC) / MDIMA)
#define KDIMB ((MDIMC * NDIMC) / NDIMB)
#define MWA (MWG / MDIMA)
#define KWA (KWG / KDIMA)
#define NWB (NWG / NDIMB)
#define KWB (KWG / KDIMB)

template <int V>
struct Vec;
template <>
struct Vec<1> {
  float v[1];
};
template <>
struct alignas(8) Vec<2> {
  float v[2];
};
template <>
struct alignas(16) Vec<4> {
  float v[4];
};
template <>
struct alignas(16) Vec<8> {
  float v[8];
};

template <int V>
__device__ __forceinline__ void ldv(float* dst, const float* src) {
  if constexpr (V == 1) {
    dst[0] = *src;
  } else if constexpr (V == 2) {
    float2 x = *reinterpret_cast<const float2*>(src);
    dst[0] = x.x;
    dst[1] = x.y;
  } else {
#pragma unroll
    for (int q = 0; q < V; q += 4) {
      float4 x = *reinterpret_cast<const float4*>(src + q);
      dst[q] = x.x;
      dst[q + 1] = x.y;
      dst[q + 2] = x.z;
      dst[q + 3] = x.w;
    }
  }
}

template <int V>
__device__ __forceinline__ void ldv_global(float* dst, const float* src) {
  if constexpr (V == 1) {
    dst[0] = __ldg(src);
  } else if constexpr (V == 2) {
    float2 x = __ldg(reinterpret_cast<const float2*>(src));
    dst[0] = x.x;
    dst[1] = x.y;
  } else {
#pragma unroll
    for (int q = 0; q < V; q += 4) {
      float4 x = __ldg(reinterpret_cast<const float4*>(src + q));
      dst[q] = x.x;
      dst[q + 1] = x.y;
      dst[q + 2] = x.z;
      dst[q + 3] = x.w;
    }
  }
}

template <int V>
__device__ __forceinline__ void stv(float* dst, const float* src) {
  if constexpr (V == 1) {
    *dst = src[0];
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(dst) = make_float2(src[0], src[1]);
  } else {
#pragma unroll
    for (int q = 0; q < V; q += 4)
      *reinterpret_cast<float4*>(dst + q) = make_float4(src[q], src[q + 1], src[q + 2], src[q + 3]);
  }
}

// vector index (within the block tile) of a thread's i-th vector
__device__ __forceinline__ constexpr int vidx_m(int i, int t) {
  return STRM ? i * MDIMC + t : t * (MWI / VWM) + i;
}
__device__ __forceinline__ constexpr int vidx_n(int i, int t) {
  return STRN ? i * NDIMC + t : t * (NWI / VWN) + i;
}

// Software pipeline (our B200 implementation choice, not a tunable): staged
// k-tiles travel global -> shared by cp.async (LDGSTS) with exactly the
// thread-to-element mapping and vector widths of the CLBlast load tunables
// (MDIMA/NDIMB re-shape, VWM/VWN widths, STRM/STRN), into a GEMM_NS-deep
// shared ring: GEMM_NS-1 k-tiles are in flight while one is consumed, no
// registers hold the prefetch (the register round trip cost ~30 registers
// per thread and capped the larger register tiles' occupancy), one barrier
// per k-tile.
#ifndef GEMM_NS
#define GEMM_NS 3
#endif

template <int V>
__device__ __forceinline__ void cp_async_vec(float* dst, const float* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if constexpr (V == 1) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
  } else if constexpr (V == 2) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < V; q += 4)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * (q / 4)), "l"(src + q) : "memory");
  }
}

extern "C" __global__ void __launch_bounds__(MDIMC * NDIMC)
gemm_kernel(float* __restrict__ C, const float* __restrict__ A, const float* __restrict__ B) {
  const int tid = threadIdx.x;
  const int tx = tid % MDIMC, ty = tid / MDIMC;
  const int m0 = blockIdx.x * MWG, n0 = blockIdx.y * NWG;
#if SA || SB
  extern __shared__ float4 gemm_smem4[];
  float* smem = reinterpret_cast<float*>(gemm_smem4);
#endif
#if SA
  float* alm = smem;  // [GEMM_NS][KWG][MWG]
  const int la0 = tid % MDIMA, la1 = tid / MDIMA;
#endif
#if SB
  float* blm = smem + (SA ? GEMM_NS * KWG * MWG : 0);  // [GEMM_NS][KWG][NWG]
  const int lb0 = tid % NDIMB, lb1 = tid / NDIMB;
#endif
  // accumulators as M-pairs: the rank-1 update of a k step is packed FFMA2
  // (a pair of A values x a broadcast B value), per component the same fmaf
  // as the scalar form -> bit-identical; odd MWI keeps a scalar last row
  float2 acc[NWI][MP];
#pragma unroll
  for (int j = 0; j < NWI; ++j)
#pragma unroll
    for (int i = 0; i < MP; ++i) acc[j][i] = make_float2(0.f, 0.f);

  // issue the async copies of k-tile `kw` into ring slot `buf`, then commit
  auto fetch = [&](int kw, int buf) {
    if (kw < GK) {
#if SA
#pragma unroll
      for (int kia = 0; kia < KWA; ++kia)
#pragma unroll
        for (int mia = 0; mia < MWA / VWM; ++mia) {
          const int mv = STRM ? mia * MDIMA + la0 : la0 * (MWA / VWM) + mia;
          cp_async_vec<VWM>(alm + buf * KWG * MWG + (kia * KDIMA + la1) * MWG + mv * VWM,
                            A + (size_t)(kw + kia * KDIMA + la1) * GM + m0 + mv * VWM);
        }
#endif
#if SB
#pragma unroll
      for (int kib = 0; kib < KWB; ++kib)
#pragma unroll
        for (int nib = 0; nib < NWB / VWN; ++nib) {
          const int nv = STRN ? nib * NDIMB + lb0 : lb0 * (NWB / VWN) + nib;
          cp_async_vec<VWN>(blm + buf * KWG * NWG + (kib * KDIMB + lb1) * NWG + nv * VWN,
                            B + (size_t)(kw + kib * KDIMB + lb1) * GN + n0 + nv * VWN);
        }
#endif
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (empty groups keep the count uniform)
  };
  (void)fetch;

#if SA || SB
#pragma unroll
  for (int s = 0; s < GEMM_NS - 1; ++s) fetch(s * KWG, s);
#endif
  int buf = 0;
  for (int kw = 0; kw < GK; kw += KWG) {
#if SA || SB
    asm volatile("cp.async.wait_group %0;" ::"n"(GEMM_NS - 2) : "memory");
    __syncthreads();  // k-tile kw visible to all; everyone is done with the slot refilled below
    fetch(kw + (GEMM_NS - 1) * KWG, (buf + GEMM_NS - 1) % GEMM_NS);
#endif
#pragma unroll
    for (int k = 0; k < KWG; ++k) {
      float a[MWI], b[NWI];
#pragma unroll
      for (int i = 0; i < MWI / VWM; ++i) {
        const int mv = vidx_m(i, tx);
#if SA
        ldv<VWM>(a + i * VWM, alm + buf * KWG * MWG + k * MWG + mv * VWM);
#else
        ldv_global<VWM>(a + i * VWM, A + (size_t)(kw + k) * GM + m0 + mv * VWM);
#endif
      }
#pragma unroll
      for (int j = 0; j < NWI / VWN; ++j) {
        const int nv = vidx_n(j, ty);
#if SB
        ldv<VWN>(b + j * VWN, blm + buf * KWG * NWG + k * NWG + nv * VWN);
#else
        ldv_global<VWN>(b + j * VWN, B + (size_t)(kw + k) * GN + n0 + nv * VWN);
#endif
      }
#pragma unroll
      for (int j = 0; j < NWI; ++j)
#pragma unroll
        for (int i = 0; i < MP; ++i) {
          if (2 * i + 1 < MWI)
            acc[j][i] = __ffma2_rn(make_float2(a[2 * i], a[2 * i + 1]), make_float2(b[j], b[j]), acc[j][i]);
          else
            acc[j][i].x = fmaf(a[2 * i], b[j], acc[j][i].x);
        }
    }
#if SA || SB
    buf = (buf + 1) % GEMM_NS;
#endif
  }
  (void)buf;

#pragma unroll
  for (int j = 0; j < NWI / VWN; ++j)
#pragma unroll
    for (int w = 0; w < VWN; ++w) {
      const int n = n0 + vidx_n(j, ty) * VWN + w;
#pragma unroll
      for (int i = 0; i < MWI / VWM; ++i) {
        const int m = m0 + vidx_m(i, tx) * VWM;
        float v[VWM];
#pragma unroll
        for (int u = 0; u < VWM; ++u) {
          const int e = i * VWM + u;
          v[u] = (e % 2 == 0) ? acc[j * VWN + w][e / 2].x : acc[j * VWN + w][e / 2].y;
        }
        stv<VWM>(C + (size_t)n * GM + m, v);
      }
    }
}

#endif  // REFERENCE_ONLY

// Naive reference: one c(m,n) per thread, sequential fmaf over k.
extern "C" __global__ void __launch_bounds__(256)
gemm_reference(float* __restrict__ C, const float* __restrict__ A, const float* __restrict__ B) {
  const int m = blockIdx.x * 64 + (threadIdx.x & 63);
  const int n = blockIdx.y * 4 + (threadIdx.x >> 6);
  if (m >= GM || n >= GN) return;
  float acc = 0.f;
  for (int k = 0; k < GK; ++k) acc = fmaf(A[(size_t)k * GM + m], B[(size_t)k * GN + n], acc);
  C[(size_t)n * GM + m] = acc;
}
