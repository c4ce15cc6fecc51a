// Per-level QTT contraction on the FP64 tensor cores of sm_100a.
//
// One launch applies one core G_k (Alg. 2 lines 5-8):
//   line 6 (column merge)  : a free view -- row m of the A operand is the 2*r_in
//                            contiguous doubles at in + 2m*r_in  (j_k-major)
//   line 7 (phi = M_k b_k) : [M x 2r_in] . [2r_in x 2r_out] on DMMA (mma.sync f64)
//   line 8 (row separation): epilogue writes output half i_k to rows
//                            m + (N/2)(s + i_k), i.e. i_k becomes the most
//                            significant column digit.
//
// Data movement (B200-first):
//   * the core (B operand) is packed on the host directly in per-lane MMA
//     fragment order and lives in shared memory for the CTA's lifetime;
//   * A tiles are contiguous row blocks, moved HBM -> smem by the TMA bulk
//     engine (cp.async.bulk + mbarrier complete_tx) in a multi-stage ring
//     filled by a dedicated producer warp;
//   * the contraction index is permuted inside each 16-wide k block
//     (logical k = t0 + 4q  <->  physical k = 4 t0 + q) so that every lane's
//     A fragment is 32 contiguous bytes (two LDS.128); the host applies the
//     same permutation to B.
#include "qtt_internal.h"

#include <cstdint>
#include <cuda_runtime.h>

namespace qtt {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
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

// D(16x8) += A(16x16) . B(16x8), fp64, fragments per the PTX ISA m16n8k16 layout.
__device__ __forceinline__ void mma_16816(double (&d)[4], const double (&a)[8], const double4& b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b.x), "d"(b.y), "d"(b.z), "d"(b.w));
}

constexpr int kBarBytes = 256;   // full[8] + empty[8] mbarriers, padded

__host__ __device__ constexpr uint32_t round_up_u32(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

template <int KB, int NB>
__global__ void __launch_bounds__((kDmmaConsumerWarps + 1) * 32, 1)
level_dmma_kernel(const LevelArgs p) {
  constexpr int CW = kDmmaConsumerWarps;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  double4* sB = reinterpret_cast<double4*>(smem + kBarBytes);
  unsigned char* sA = smem + kBarBytes + KB * NB * 32 * sizeof(double4);

  const int K = p.K;
  const int S = p.stages;
  const int rows_per_stage = kDmmaRowsPerSubtile * p.rep;
  const uint32_t stage_stride = round_up_u32(uint32_t(rows_per_stage) * uint32_t(K) * 8u, 128u);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // B operand (the packed core) -> smem, once per CTA.
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
  __syncthreads();

  const int64_t M = p.M;
  const int64_t nstage_tiles = (M + rows_per_stage - 1) / rows_per_stage;

  if (warp == CW) {
    // ---------------- TMA producer (one lane) ----------------
    if (lane == 0) {
      int it = 0;
      for (int64_t t = blockIdx.x; t < nstage_tiles; t += gridDim.x, ++it) {
        const int s = it % S;
        const uint32_t ph = uint32_t(it / S) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        const int64_t m0 = t * rows_per_stage;
        const int64_t rows = (M - m0) < rows_per_stage ? (M - m0) : rows_per_stage;
        const uint32_t bytes = uint32_t(rows) * uint32_t(K) * 8u;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(sA + size_t(s) * stage_stride, p.in + m0 * K, bytes, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers: 4 warps x 16 rows per sub-tile ----------------
  const int g = lane >> 2;
  const int t0 = lane & 3;
  const bool kfull = (K == 16 * KB);
  const bool vec_out = (p.r_out % 2) == 0;
  const int RP = p.RP;
  const int r_out = p.r_out;
  const int64_t half = p.half;

  int it = 0;
  for (int64_t t = blockIdx.x; t < nstage_tiles; t += gridDim.x, ++it) {
    const int s = it % S;
    const uint32_t ph = uint32_t(it / S) & 1u;
    mbar_wait(&full[s], ph);
    const double* stage = reinterpret_cast<const double*>(sA + size_t(s) * stage_stride);
    const int64_t m_stage = t * rows_per_stage;

    for (int u = 0; u < p.rep; ++u) {
      const int lrow = u * kDmmaRowsPerSubtile + warp * 16 + g;     // local row of this lane (h = 0)
      const double* r0 = stage + size_t(lrow) * K;
      const double* r1 = r0 + size_t(8) * K;
      double c[NB][4];
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) c[nb][0] = c[nb][1] = c[nb][2] = c[nb][3] = 0.0;
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        double a[8];
        const int kbase = kb * 16 + 4 * t0;
        if (kfull || kb < KB - 1) {
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
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const double4 b = sB[(kb * NB + nb) * 32 + lane];
          mma_16816(c[nb], a, b);
        }
      }
      if (u == p.rep - 1) {
        // all smem reads of this stage are complete (their values were consumed above)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // ---- epilogue: row separation (Alg. 2 line 8) ----
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t m = m_stage + lrow + 8 * h;
        if (m >= M) continue;
        const int64_t sr = m / half;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const int n = nb * 8 + 2 * t0;
          const int i = n / RP;
          const int b = n - i * RP;
          if (i > 1 || b >= r_out) continue;
          double* dst = p.out + (m + half * (sr + i)) * r_out + b;
          const double v0 = c[nb][2 * h], v1 = c[nb][2 * h + 1];
          if (vec_out) {
            *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
          } else {
            dst[0] = v0;
            if (b + 1 < r_out) dst[1] = v1;
          }
        }
      }
    }
  }
}

using KernelFn = void (*)(const LevelArgs);

template <int KB, int NB>
constexpr KernelFn kfn() { return &level_dmma_kernel<KB, NB>; }

#define QTT_ROW(KB)                                                                                 \
  {kfn<KB, 1>(), kfn<KB, 2>(), kfn<KB, 3>(), kfn<KB, 4>(), kfn<KB, 5>(), kfn<KB, 6>(), kfn<KB, 7>(), \
   kfn<KB, 8>(), kfn<KB, 9>(), kfn<KB, 10>(), kfn<KB, 11>(), kfn<KB, 12>()}

const KernelFn kTable[kMaxKB][kMaxNB] = {QTT_ROW(1), QTT_ROW(2), QTT_ROW(3), QTT_ROW(4), QTT_ROW(5), QTT_ROW(6)};

KernelFn lookup(int KB, int NB) {
  if (KB < 1 || KB > kMaxKB || NB < 1 || NB > kMaxNB) return nullptr;
  return kTable[KB - 1][NB - 1];
}

// ---------------------------------------------------------------------------
// Generic level kernel (any rank): one thread per output element.  Slow but
// simple; used for ranks above the DMMA instantiations.
// ---------------------------------------------------------------------------
__global__ void level_generic_kernel(const LevelArgs p) {
  const int r_in = p.r_in, r_out = p.r_out;
  const int64_t total = p.M * 2 * r_out;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = idx / (2 * r_out);
    const int rem = int(idx - m * 2 * r_out);
    const int i = rem / r_out;
    const int b = rem - i * r_out;
    double acc = 0.0;
    for (int j = 0; j < 2; ++j) {
      const double* in = p.in + (2 * m + j) * r_in;
      const double* g = p.core + (size_t(i) * 2 + j) * r_out + b;   // G[a][i][j][b], a stride 4 r_out
      for (int a = 0; a < r_in; ++a) acc = fma(g[size_t(a) * 4 * r_out], in[a], acc);
    }
    const int64_t sr = m / p.half;
    p.out[(m + p.half * (sr + i)) * r_out + b] = acc;
  }
}

}  // namespace

size_t dmma_smem_bytes(int KB, int NB, int K, int rep, int stages) {
  const size_t stage = round_up_u32(uint32_t(kDmmaRowsPerSubtile * rep) * uint32_t(K) * 8u, 128u);
  return kBarBytes + size_t(KB) * NB * 32 * sizeof(double4) + stage * stages;
}

cudaError_t dmma_prepare(int KB, int NB, size_t smem) {
  KernelFn f = lookup(KB, NB);
  if (!f) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              int(smem));
}

cudaError_t dmma_occupancy(int KB, int NB, size_t smem, int* ctas_per_sm) {
  KernelFn f = lookup(KB, NB);
  if (!f) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, reinterpret_cast<const void*>(f),
                                                       (kDmmaConsumerWarps + 1) * 32, smem);
}

cudaError_t launch_level_dmma(const LevelArgs& a, cudaStream_t st) {
  KernelFn f = lookup(a.KB, a.NB);
  if (!f) return cudaErrorInvalidValue;
  f<<<a.grid, (kDmmaConsumerWarps + 1) * 32, a.smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_level_generic(const LevelArgs& a, cudaStream_t st, int num_sms) {
  const int64_t total = a.M * 2 * a.r_out;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = int64_t(num_sms) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  level_generic_kernel<<<int(blocks), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace qtt
