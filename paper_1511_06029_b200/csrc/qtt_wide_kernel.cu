// Wide merged stage: the super-core W of L consecutive levels (qtt_plan.cpp) is
// applied as one DMMA GEMM  C[M x Nout] = A[M x K] . W[K x Nout]  whose W is too
// large for shared memory (K = 2^L r_in and Nout = 2^L r_out up to thousands).
//
// Where it pays (Alg. 2, costs 4 r_{k-1} r_k flops per
// element per level): at the ends of a rank profile (r_0 = r_d = 1) the
// product of the first (last) L cores is a dense 2^L r_L x 2^L matrix whose
// application costs 2^(L+1) r_L flops per element -- 12288 for c4's levels
// 1..7 (r_7 = 48) against Alg. 2's 18088 -- and none of the L-1 intermediates
// ever reaches HBM.  The product is the QTT definition itself
// restricted to those digits, so the result is exact up to fp64 rounding.
//
// Structure (persistent, one CTA per SM, (4*CG + 1) warps):
//   * tile = 64 rows x (8*NB) columns of C; a dynamic scheduler (atomicAdd)
//     hands out tiles column-block-minor, so CTAs running at the same time
//     share A row tiles in L2;
//   * producer warp: per k-chunk of 32, the A chunk (64 row segments of 256 B,
//     one cp.async.bulk each, issued by the 32 lanes, into rows padded to 34
//     doubles so the A fragment loads are bank-conflict free) and the W chunk
//     (one contiguous cp.async.bulk of fragment-packed doubles, 8-32 KiB,
//     L2-resident across tiles) land in a 4-stage mbarrier ring;
//   * 4 x CG consumer warps accumulate over all k-chunks of a tile in
//     registers (DMMA m8n8k4, as in qtt_dmma_kernel.cuh) and store with the
//     row-separation epilogue of the stage (out row m + Q*(s*(2^L-1) + ii)).
#include "qtt_dmma_kernel.cuh"

#include <cstdint>
#include <cuda_runtime.h>

namespace qtt {
namespace wide {
namespace {

using dmma::bulk_g2s;
using dmma::dmma_884;
using dmma::fence_mbar_init;
using dmma::load_a16;
using dmma::mbar_arrive;
using dmma::mbar_arrive_expect_tx;
using dmma::mbar_init;
using dmma::mbar_wait;

constexpr uint32_t kAStageBytes = uint32_t(kDmmaRowsPerSubtile) * kWideSA * 8;   // 17408
__host__ __device__ constexpr uint32_t b_chunk_bytes(int NB) { return uint32_t(kWideKBC) * NB * 32 * 32; }
__host__ __device__ constexpr uint32_t stage_bytes(int NB) { return kAStageBytes + b_chunk_bytes(NB); }

// Accumulate one k-chunk (kWideKBC k16 blocks) into c: 16 rows x NBC n8-blocks.
template <int NB, int NBC>
__device__ __forceinline__ void chunk_mma(double (&c)[NBC][4], const double* r0, const double* r1,
                                          const double4* sB, int nb0, int lane) {
  const int t0 = lane & 3;
#pragma unroll
  for (int kb = 0; kb < kWideKBC; ++kb) {
    double a[8];
    load_a16<true>(a, r0, r1, kb * 16 + 4 * t0, kWideBK);
    double4 b[NBC];
#pragma unroll
    for (int nb = 0; nb < NBC; ++nb) b[nb] = sB[(kb * NB + nb0 + nb) * 32 + lane];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int nb = 0; nb < NBC; ++nb) {
        const double bq = q == 0 ? b[nb].x : q == 1 ? b[nb].y : q == 2 ? b[nb].z : b[nb].w;
        dmma_884(c[nb][0], c[nb][1], a[2 * q], bq);
        dmma_884(c[nb][2], c[nb][3], a[2 * q + 1], bq);
      }
    }
  }
}

// Row-separation epilogue (Alg. 2 line 8 for all L levels): column n = ii*r_out + b
// of GEMM row m goes to out[(m + Q*(s*(n_i-1) + ii)) * r_out + b], s = m / Q.
template <int NBC>
__device__ __forceinline__ void tile_store(const double (&c)[NBC][4], const LevelArgs& p, int64_t m_first,
                                           int n_first, int lane) {
  const int g = lane >> 2, t0 = lane & 3;
  const int r_out = p.r_out;
  const bool vec = (r_out % 2) == 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t m = m_first + g + 8 * h;
    if (m >= p.M) continue;
    const int64_t rowbase = m + (((m >> p.log2_q) * (p.n_i - 1)) << p.log2_q);
#pragma unroll
    for (int nb = 0; nb < NBC; ++nb) {
      const int n = n_first + nb * 8 + 2 * t0;
      if (n >= p.nout) continue;
      const int ii = n / r_out;
      const int b = n - ii * r_out;
      double* dst = p.out + (rowbase + (int64_t(ii) << p.log2_q)) * r_out + b;
      if (vec) {
        *reinterpret_cast<double2*>(dst) = make_double2(c[nb][2 * h], c[nb][2 * h + 1]);
      } else {
        dst[0] = c[nb][2 * h];
        const int n1 = n + 1;
        if (n1 < p.nout) {
          const int ii1 = n1 / r_out;
          const int b1 = n1 - ii1 * r_out;
          p.out[(rowbase + (int64_t(ii1) << p.log2_q)) * r_out + b1] = c[nb][2 * h + 1];
        }
      }
    }
  }
}

template <int NB, int NBC>
__device__ __forceinline__ void consumer(const LevelArgs& p, uint64_t* full, uint64_t* empty, const int64_t* tile_id,
                                         unsigned char* ring, int rg, int nb0, int lane) {
  const int g = lane >> 2;
  double c[NBC][4];
  int chunk = 0;
  for (int it = 0;; ++it) {
    const int s = it % kWideStages;
    const uint32_t ph = uint32_t(it / kWideStages) & 1u;
    mbar_wait(&full[s], ph);
    const int64_t t = tile_id[s];
    if (t < 0) break;
    if (chunk == 0) {
#pragma unroll
      for (int nb = 0; nb < NBC; ++nb) c[nb][0] = c[nb][1] = c[nb][2] = c[nb][3] = 0.0;
    }
    const unsigned char* st = ring + size_t(s) * stage_bytes(NB);
    const double* r0 = reinterpret_cast<const double*>(st) + size_t(rg * 16 + g) * kWideSA;
    const double* r1 = r0 + 8 * kWideSA;
    chunk_mma<NB, NBC>(c, r0, r1, reinterpret_cast<const double4*>(st + kAStageBytes), nb0, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++chunk == p.nchunks) {
      chunk = 0;
      const int64_t rt = t / p.ncb;
      const int cb = int(t - rt * p.ncb);
      tile_store<NBC>(c, p, rt * kDmmaRowsPerSubtile + rg * 16, (cb * NB + nb0) * 8, lane);
    }
  }
}

template <int NB>
__global__ void __launch_bounds__(dmma_threads(NB), 1) wide_dmma_kernel(const LevelArgs p) {
  constexpr int CG = dmma_col_groups(NB);
  constexpr int CW = kDmmaRowGroups * CG;
  constexpr int NBW = (NB + CG - 1) / CG;
  constexpr int NB_1 = (NB - NBW) < NBW ? (NB - NBW) : NBW;
  constexpr int NB_2 = NB - NBW - NB_1;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  int64_t* tile_id = reinterpret_cast<int64_t*>(empty + kMaxStages);
  unsigned char* ring = smem + kBarBytes;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWideStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == CW) {
    // ---------------- producer warp: tile scheduler + TMA bulk loads ----------------
    const int64_t M = p.M;
    const int64_t K = p.K;
    const int64_t ntiles = ((M + kDmmaRowsPerSubtile - 1) / kDmmaRowsPerSubtile) * p.ncb;
    const uint32_t bbytes = b_chunk_bytes(NB);
    int it = 0;
    for (;;) {
      int64_t t = 0;
      if (lane == 0) t = atomicAdd(p.tile_counter, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntiles) {
        const int s = it % kWideStages;
        mbar_wait(&empty[s], (uint32_t(it / kWideStages) & 1u) ^ 1u);
        if (lane == 0) {
          tile_id[s] = -1;
          mbar_arrive(&full[s]);
        }
        break;
      }
      const int64_t rt = t / p.ncb;
      const int cb = int(t - rt * p.ncb);
      const int64_t m0 = rt * kDmmaRowsPerSubtile;
      const int rows = int((M - m0) < kDmmaRowsPerSubtile ? (M - m0) : kDmmaRowsPerSubtile);
      const double* arow = p.in + m0 * K;
      const double* bsrc = p.bpack + size_t(cb) * p.nchunks * (bbytes / 8);
      for (int ch = 0; ch < p.nchunks; ++ch, ++it) {
        const int s = it % kWideStages;
        mbar_wait(&empty[s], (uint32_t(it / kWideStages) & 1u) ^ 1u);
        unsigned char* st = ring + size_t(s) * stage_bytes(NB);
        if (lane == 0) {
          tile_id[s] = t;
          mbar_arrive_expect_tx(&full[s], uint32_t(rows) * kWideBK * 8u + bbytes);
          bulk_g2s(st + kAStageBytes, bsrc + size_t(ch) * (bbytes / 8), bbytes, &full[s]);
        }
        __syncwarp();
        for (int r = lane; r < rows; r += 32)
          bulk_g2s(st + size_t(r) * kWideSA * 8, arow + r * K + ch * kWideBK, kWideBK * 8, &full[s]);
      }
    }
    return;
  }
  const int rg = warp % kDmmaRowGroups;
  const int cg = warp / kDmmaRowGroups;
  if (cg == 0) {
    consumer<NB, NBW>(p, full, empty, tile_id, ring, rg, 0, lane);
  } else if (cg == 1) {
    if constexpr (NB_1 > 0) consumer<NB, NB_1>(p, full, empty, tile_id, ring, rg, NBW, lane);
  } else {
    if constexpr (NB_2 > 0) consumer<NB, NB_2>(p, full, empty, tile_id, ring, rg, NBW + NB_1, lane);
  }
}

using KernelFn = void (*)(const LevelArgs);

KernelFn lookup(int NB) {
  switch (NB) {
    case 4: return &wide_dmma_kernel<4>;
    case 8: return &wide_dmma_kernel<8>;
    case 12: return &wide_dmma_kernel<12>;
    case 16: return &wide_dmma_kernel<16>;
    default: return nullptr;
  }
}

}  // namespace
}  // namespace wide

size_t wide_smem_bytes(int NB) { return kBarBytes + size_t(kWideStages) * wide::stage_bytes(NB); }

cudaError_t wide_prepare(int NB, size_t smem) {
  wide::KernelFn f = wide::lookup(NB);
  if (!f) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              int(smem));
}

cudaError_t launch_wide(const LevelArgs& a, cudaStream_t st) {
  wide::KernelFn f = wide::lookup(a.NB);
  if (!f) return cudaErrorInvalidValue;
  f<<<a.grid, dmma_threads(a.NB), a.smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace qtt
