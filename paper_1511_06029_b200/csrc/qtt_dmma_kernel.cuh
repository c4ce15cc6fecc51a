// DMMA stage kernel template (Alg. 2 lines 5-8), shared by
// the instantiation units qtt_dmma_inst*.cu.  See qtt_level_dmma.cu for the design.
#pragma once
#include "qtt_internal.h"

#include <cstdint>
#include <cuda_runtime.h>

namespace qtt {
namespace dmma {
namespace {   // each instantiation unit gets its own internal copy

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// Programmatic dependent launch.  Every stage kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so its launch is
// processed while the previous kernel on the stream runs; pdl_wait() (before
// the first access to any buffer another kernel writes or reads: activations,
// tile counters, split scratch, flags) blocks until the previous kernel has
// completed.  Only static operands (the packed cores) are read before it.  No
// kernel issues griddepcontrol.launch_dependents (the implicit trigger at CTA
// exit): an early trigger when a CTA's scheduler runs dry measured no gain
// (c1-c3 within 1%).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion signalled on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__host__ __device__ constexpr uint32_t round_up_u32(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// One 8x8x4 fp64 MMA (the native DMMA shape): d(8x8) += a(8x4) . b(4x8).
// Fragments: a = A[g][t0], b = B[t0][g], d = {D[g][2 t0], D[g][2 t0 + 1]}
// with g = lane / 4, t0 = lane % 4.
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// A fragments of one 16-row x 16-k block for this lane: a[2q + h] is the
// value of k4-step q for row half h (rows g and g + 8), i.e. physical
// column 4*t0 + q of rows r0 (h = 0) and r1 (h = 1).
template <bool FULL>
__device__ __forceinline__ void load_a16(double (&a)[8], const double* r0, const double* r1, int kbase, int K) {
  if (FULL) {
    const double2 x0 = *reinterpret_cast<const double2*>(r0 + kbase);
    const double2 x1 = *reinterpret_cast<const double2*>(r0 + kbase + 2);
    const double2 y0 = *reinterpret_cast<const double2*>(r1 + kbase);
    const double2 y1 = *reinterpret_cast<const double2*>(r1 + kbase + 2);
    a[0] = x0.x; a[2] = x0.y; a[4] = x1.x; a[6] = x1.y;
    a[1] = y0.x; a[3] = y0.y; a[5] = y1.x; a[7] = y1.y;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool ok = (kbase + q) < K;
      a[2 * q] = ok ? r0[kbase + q] : 0.0;
      a[2 * q + 1] = ok ? r1[kbase + q] : 0.0;
    }
  }
}

// 16 rows x NBC n8-blocks (starting at n-block nb0) of one sub-tile:
// c[nb][2h + v] = D[row g + 8h][col (nb0+nb)*8 + 2 t0 + v].
// Issue order: k4-step outermost, then n-block, then row half, so that two
// DMMAs into the same accumulator are 2*NBC instructions apart.
template <int KB, int NB, int NBC>
__device__ __forceinline__ void subtile_mma(double (&c)[NBC > 0 ? NBC : 1][4], const double* r0, const double* r1,
                                            const double4* sB, int nb0, int lane, int K, bool kfull) {
  const int t0 = lane & 3;
#pragma unroll
  for (int nb = 0; nb < NBC; ++nb) c[nb][0] = c[nb][1] = c[nb][2] = c[nb][3] = 0.0;
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
    double a[8];
    const int kbase = kb * 16 + 4 * t0;
    if (kfull || kb < KB - 1) load_a16<true>(a, r0, r1, kbase, K);
    else load_a16<false>(a, r0, r1, kbase, K);
    double4 b[NBC > 0 ? NBC : 1];
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

// Alg. 2 line 8 (row separation), applied for all L levels of the stage at
// once: column n = ii*RP + b of GEMM row m goes to out row
// m + Q*(s*(n_i-1) + ii), s = m / Q (the RHS index; Q = N / n_i is a power of 2).
// coff[nb] = Q*ii*r_out + b for this lane's column pair, or -1 if padding.
template <int NBC>
__device__ __forceinline__ void subtile_store(const double (&c)[NBC > 0 ? NBC : 1][4], const LevelArgs& p,
                                              const int64_t (&coff)[NBC > 0 ? NBC : 1], bool vec_out,
                                              int64_t m_first, int lane) {
  const int g = lane >> 2;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t m = m_first + g + 8 * h;
    if (m >= p.M) continue;
    double* rowp = p.out + (m + (((m >> p.log2_q) * (p.n_i - 1)) << p.log2_q)) * p.r_out;
#pragma unroll
    for (int nb = 0; nb < NBC; ++nb) {
      if (coff[nb] < 0) continue;
      double* dst = rowp + coff[nb];
      const double v0 = c[nb][2 * h], v1 = c[nb][2 * h + 1];
      QTT_CHECK_OUT(p, dst, vec_out ? 2 : 1);
      if (vec_out) {
        *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
      } else {
        dst[0] = v0;
        if (((coff[nb] % p.r_out) + 1) < p.r_out) dst[1] = v1;
      }
    }
  }
}

// Consumer loop of one warp: row group rg (16 rows of each 64-row sub-tile),
// n-blocks [nb0, nb0 + NBC).  Tiles arrive from the producer through the
// smem ring; tile index -1 ends the loop.
template <int KB, int NB, int NBC>
__device__ __forceinline__ void consumer_loop(const LevelArgs& p, uint64_t* full, uint64_t* empty,
                                              const int64_t* tile_id, const double4* sB,
                                              const unsigned char* sA, uint32_t stage_stride, int rg, int nb0,
                                              int lane) {
  const int K = p.K;
  const int S = p.stages;
  const int rows_per_stage = kDmmaRowsPerSubtile * p.rep;
  const bool kfull = (K == 16 * KB);
  const bool vec_out = (p.r_out % 2) == 0;
  const int g = lane >> 2, t0 = lane & 3;
  int64_t coff[NBC > 0 ? NBC : 1];
#pragma unroll
  for (int nb = 0; nb < NBC; ++nb) {
    const int n = (nb0 + nb) * 8 + 2 * t0;
    const int i = n / p.RP;
    const int b = n - i * p.RP;
    coff[nb] = (i >= p.n_i || b >= p.r_out) ? int64_t(-1) : ((int64_t(i) << p.log2_q) * p.r_out + b);
  }
  // ring stage and phase kept as counters: `it % S`, `it / S` with the runtime
  // S cost a ~35-instruction reciprocal sequence in front of every tile's
  // barrier wait (ncu source page), which the warps of a sub-partition run together
  int s = 0;
  uint32_t ph = 0;
  for (;; ++s) {
    if (s == S) {
      s = 0;
      ph ^= 1u;
    }
    mbar_wait(&full[s], ph);
    const int64_t t = tile_id[s];
    if (t < 0) break;
    const double* stage = reinterpret_cast<const double*>(sA + size_t(s) * stage_stride);
    const int64_t m_stage = t * rows_per_stage;
    for (int u = 0; u < p.rep; ++u) {
      const int lrow0 = u * kDmmaRowsPerSubtile + rg * 16;
      const double* r0 = stage + size_t(lrow0 + g) * K;
      const double* r1 = r0 + size_t(8) * K;
      double c[NBC > 0 ? NBC : 1][4];
      if (NBC > 0) subtile_mma<KB, NB, NBC>(c, r0, r1, sB, nb0, lane, K, kfull);
      if (u == p.rep - 1) {
        // every smem read of this stage has been consumed by the MMAs above
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (NBC > 0) subtile_store<NBC>(c, p, coff, vec_out, m_stage + lrow0, lane);
    }
  }
}

template <int KB, int NB>
__global__ void __launch_bounds__(dmma_threads(NB), 1)
level_dmma_kernel(const LevelArgs p) {
  constexpr int CG = dmma_col_groups(NB);
  constexpr int CW = kDmmaRowGroups * CG;         // consumer warps
#ifdef QTT_UNEVEN_CG
  // experiment: unequal column groups, so the warps of a sub-partition reach
  // their epilogues at different times
  constexpr int NBW = (NB + CG - 1) / CG + ((CG >= 2 && NB >= 2 * CG) ? 1 : 0);
  constexpr int NB_1 = CG == 1 ? 0 : CG == 2 ? NB - NBW : (NB - NBW + 1) / 2 + (((NB - NBW) % 2 == 0) ? 1 : 0);
  constexpr int NB_2 = NB - NBW - NB_1;
  static_assert(NB_1 >= 0 && NB_2 >= 0, "split");
#else
  constexpr int NBW = (NB + CG - 1) / CG;         // n-blocks per column group
  constexpr int NB_1 = (NB - NBW) < NBW ? (NB - NBW) : NBW;
  constexpr int NB_2 = NB - NBW - NB_1;
#endif
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  int64_t* tile_id = reinterpret_cast<int64_t*>(empty + kMaxStages);
  double4* sB = reinterpret_cast<double4*>(smem + kBarBytes);
  unsigned char* sA = smem + kBarBytes + KB * NB * 32 * sizeof(double4);

  const int K = p.K;
  const int S = p.stages;
  const int rows_per_stage = kDmmaRowsPerSubtile * p.rep;
  const uint32_t stage_stride = round_up_u32(uint32_t(rows_per_stage) * uint32_t(K) * 8u, 128u);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // B operand (the packed core) -> smem, once per CTA.  Read before pdl_wait():
  // bpack is written once at qtt_create, never by a kernel on the stream.
  {
    const double4* gB = reinterpret_cast<const double4*>(p.bpack);
    for (int i = threadIdx.x; i < KB * NB * 32; i += blockDim.x) sB[i] = gB[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  pdl_wait();
  __syncthreads();

  if (warp == CW) {
    // ---------------- producer: dynamic tile scheduler + TMA bulk loads ----------------
    if (lane == 0) {
      const int64_t M = p.M;
      const int64_t nstage_tiles = (M + rows_per_stage - 1) / rows_per_stage;
      int s = 0;
      uint32_t ph = 0;
      bool first = true;
      for (;; ++s) {
        if (s == S) {
          s = 0;
          ph ^= 1u;
        }
        mbar_wait(&empty[s], ph ^ 1u);
        // the first tile is the CTA's own index (grid <= tiles): no L2 atomic, with every
        // producer of the grid queueing on one address, in front of the first load
        const int64_t t = first ? int64_t(blockIdx.x) : int64_t(gridDim.x) + atomicAdd(p.tile_counter, 1);
        first = false;
        if (t >= nstage_tiles) {
          tile_id[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        tile_id[s] = t;
        const int64_t m0 = t * rows_per_stage;
        const int64_t rows = (M - m0) < rows_per_stage ? (M - m0) : rows_per_stage;
        const uint32_t bytes = uint32_t(rows) * uint32_t(K) * 8u;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(sA + size_t(s) * stage_stride, p.in + m0 * K, bytes, &full[s]);
      }
    }
    return;
  }
  const int rg = warp % kDmmaRowGroups;
  const int cg = warp / kDmmaRowGroups;
  if (cg == 0) consumer_loop<KB, NB, NBW>(p, full, empty, tile_id, sB, sA, stage_stride, rg, 0, lane);
  else if (cg == 1) consumer_loop<KB, NB, NB_1>(p, full, empty, tile_id, sB, sA, stage_stride, rg, NBW, lane);
  else consumer_loop<KB, NB, NB_2>(p, full, empty, tile_id, sB, sA, stage_stride, rg, NBW + NB_1, lane);
}

}  // namespace

using KernelFn = void (*)(const LevelArgs);

// lookup of the instances one unit holds (nullptr if not there)
KernelFn lookup_kb12(int KB, int NB);
KernelFn lookup_kb34(int KB, int NB);
KernelFn lookup_kb56(int KB, int NB);
KernelFn lookup_kb78(int KB, int NB);

}  // namespace dmma
}  // namespace qtt
