// QTT stage contraction on the FP64 tensor cores of sm_100a: host-side glue
// (instance lookup, launch), the generic fallback kernel and the diagonal-
// stage kernel (block-diagonal digits).  The DMMA kernel
// template is in qtt_dmma_kernel.cuh, instantiated by qtt_dmma_inst_kb*.cu.
//
// One launch applies one core G_k (Alg. 2 lines 5-8), or
// the super-core W of L consecutive levels (variant kMerged), as one GEMM:
//   line 6 (column merge)  : a free view -- row m of the A operand is the 2*r_in
//                            contiguous doubles at in + 2m*r_in  (j_k-major)
//   line 7 (phi = M_k b_k) : [M x 2r_in] . [2r_in x 2r_out] on DMMA (mma.sync f64)
//   line 8 (row separation): epilogue writes output half i_k to rows
//                            m + (N/2)(s + i_k), i.e. i_k becomes the most
//                            significant column digit (for a merged stage
//                            the L output digits ii go to rows
//                            m + Q*(s*(2^L-1) + ii), Q = N/2^L).
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
#include "qtt_dmma_kernel.cuh"

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace qtt {
namespace {

using dmma::KernelFn;

KernelFn lookup(int KB, int NB) {
  if (!dmma_instantiated(KB, NB)) return nullptr;
  if (KB <= 2) return dmma::lookup_kb12(KB, NB);
  if (KB <= 4) return dmma::lookup_kb34(KB, NB);
  if (KB <= 6) return dmma::lookup_kb56(KB, NB);
  return dmma::lookup_kb78(KB, NB);
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
    const int64_t sr = m >> p.log2_q;   // L = 1: n_i = 2, Q = N/2
    double* dst = p.out + (m + ((sr + i) << p.log2_q)) * r_out + b;
    QTT_CHECK_OUT(p, dst, 1);
    *dst = acc;
  }
}

// Diagonal stage (kDiag): a warp takes 32 consecutive GEMM rows m (one per
// lane) of one digit combination ii; lane m reads its input row R = m n_i + ii
// (r_in contiguous doubles, 16-byte loads, all issued before the FMAs) and
// forms the r_out <= 8 dot products with D[ii] (the same for the whole warp:
// broadcast loads).  Consecutive warps take consecutive ii, i.e. adjacent
// input rows; the 32 lanes store 32 consecutive output rows
// m + Q (s (n_i - 1) + ii).  Fixed summation order a = 0..r_in-1: deterministic.
// Measured on the BIE factor's levels 10-21 (r_in 50, 2^21 rows): 0.34 ms; a
// warp per row with shuffle reductions 0.82, each warp's 32 adjacent rows
// staged in smem (lanes then over different ii) 0.77, all row loads hoisted
// into registers 0.51.
constexpr int kDiagMaxRin = 64;
#ifndef QTT_DIAG_UNROLL
#define QTT_DIAG_UNROLL 4
#endif
constexpr int kDiagUnroll = QTT_DIAG_UNROLL;   // 16-byte row loads in flight per lane

// LANE_II (few GEMM rows, M < 32, e.g. a diagonal matrix: one stage of all d
// levels, M = nrhs): lanes take 32 consecutive ii of one m instead.
template <bool VEC, bool LANE_II>
__global__ void __launch_bounds__(256) diag_kernel(const LevelArgs p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int r_in = p.r_in, r_out = p.r_out, n_i = p.n_i;
  const int64_t mblocks = LANE_II ? p.M : (p.M + 31) / 32;
  const int64_t items = LANE_II ? mblocks * ((n_i + 31) / 32) : mblocks * n_i;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    int64_t m;
    int ii;
    if (LANE_II) {
      const int iblocks = (n_i + 31) / 32;
      m = w / iblocks;
      ii = int(w - m * iblocks) * 32 + lane;
      if (ii >= n_i) continue;
    } else {
      const int64_t mb = w / n_i;
      ii = int(w - mb * n_i);
      m = mb * 32 + lane;
      if (m >= p.M) continue;
    }
    const double* x = p.in + (m * n_i + ii) * r_in;
    const double* D = p.core + size_t(ii) * r_in * r_out;
    double acc[kDiagMaxROut];
#pragma unroll
    for (int b = 0; b < kDiagMaxROut; ++b) acc[b] = 0.0;
    if (VEC) {
#pragma unroll (kDiagUnroll)
      for (int a = 0; a < r_in; a += 2) {
        const double2 xa = __ldcs(reinterpret_cast<const double2*>(x + a));
#pragma unroll
        for (int b = 0; b < kDiagMaxROut; ++b)
          if (b < r_out) {
            acc[b] = fma(xa.x, __ldg(D + size_t(a) * r_out + b), acc[b]);
            acc[b] = fma(xa.y, __ldg(D + size_t(a + 1) * r_out + b), acc[b]);
          }
      }
    } else {
#pragma unroll 4
      for (int a = 0; a < r_in; ++a) {
        const double xa = __ldcs(x + a);
#pragma unroll
        for (int b = 0; b < kDiagMaxROut; ++b)
          if (b < r_out) acc[b] = fma(xa, __ldg(D + size_t(a) * r_out + b), acc[b]);
      }
    }
    const int64_t row = m + (((m >> p.log2_q) * (n_i - 1)) << p.log2_q) + (int64_t(ii) << p.log2_q);
#pragma unroll
    for (int b = 0; b < kDiagMaxROut; ++b)
      if (b < r_out) {
        QTT_CHECK_OUT(p, p.out + row * r_out + b, 1);
        p.out[row * r_out + b] = acc[b];
      }
  }
}

// Diagonal stage with r_out > 8 (e.g. block-diagonal digits at the bottom of
// a profile, r_in small): one warp per input row R, lanes over the output
// index b (two per lane, r_out <= 64); the row's r_in values are broadcast
// loads, D[ii][a][b] and the output row are coalesced.  Fixed order over a.
__global__ void __launch_bounds__(256) diag_out_kernel(const LevelArgs p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int r_in = p.r_in, r_out = p.r_out, n_i = p.n_i;
  const int64_t nrows = p.M * n_i;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t R = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; R < nrows; R += nw) {
    const int64_t m = R / n_i;
    const int ii = int(R - m * n_i);
    const double* x = p.in + R * r_in;
    const double* D = p.core + size_t(ii) * r_in * r_out;
    double acc0 = 0.0, acc1 = 0.0;
    const bool b0 = lane < r_out, b1 = lane + 32 < r_out;
#pragma unroll 4
    for (int a = 0; a < r_in; ++a) {
      const double xa = __ldg(x + a);
      if (b0) acc0 = fma(xa, __ldg(D + size_t(a) * r_out + lane), acc0);
      if (b1) acc1 = fma(xa, __ldg(D + size_t(a) * r_out + lane + 32), acc1);
    }
    const int64_t row = m + (((m >> p.log2_q) * (n_i - 1)) << p.log2_q) + (int64_t(ii) << p.log2_q);
    if (b0) {
      QTT_CHECK_OUT(p, p.out + row * r_out + lane, 1);
      p.out[row * r_out + lane] = acc0;
    }
    if (b1) {
      QTT_CHECK_OUT(p, p.out + row * r_out + lane + 32, 1);
      p.out[row * r_out + lane + 32] = acc1;
    }
  }
}

// Diagonal stage, streaming form (n_i >= kDiagChunk): a work item is CR =
// kDiagChunk (128) consecutive input rows of one GEMM row m, i.e. the digit
// combinations ii of one block ib (rows m n_i + ib CR .. + CR - 1): one
// contiguous run of x, moved HBM -> smem by one TMA bulk copy, kDiagStages
// (3) items in flight per CTA.  The items are ordered ii-block-major and each
// persistent CTA takes a contiguous range of them, so its D block (D[ii] for
// the CR ii of the block: also contiguous, one bulk copy) stays in smem
// across many m and is reloaded only when the block changes.  Two threads
// per row: thread h sums a = h, h + 2, ... (fixed order), the pair adds its
// halves with one shuffle (commutative: both hold the same sum), the even
// thread stores the row's r_out outputs (one of the 2^L output streams per ii).
// The kernel is instantiated per r_out (1..8) so its inner loop carries no
// predicates.  (Measured on the BIE factor M's levels 10-21, r_in 50, 2^21
// rows: 0.145 ms = 5.9 TB/s, 91% of the measured HBM peak, against 0.34 ms
// for diag_kernel; with r_out a runtime bound of a predicated 8-wide loop
// 0.213 ms (41% issue-active: instruction-bound); 64-row items with 6 in
// flight 0.35 ms; a warp per row with lanes over a, D from L2, 2.1 ms; a
// producer warp with full/empty mbarriers instead of the CTA barrier per item
// 0.220 ms.)
constexpr int kDiagChunk = 128;
constexpr int kDiagStages = 3;
constexpr size_t kDiagStreamSmem = 220 * 1024;

template <int RO>   // r_out, exact: the inner loops carry no predicates
__global__ void __launch_bounds__(256) diag_stream_kernel(const LevelArgs p) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kDiagStages];
  __shared__ __align__(8) uint64_t dbar;
  const int r_in = p.r_in, r_out = p.r_out, n_i = p.n_i;
  const int nblk = n_i / kDiagChunk;                                  // ii blocks
  const int64_t items = int64_t(nblk) * p.M;                          // (ib, m), ib-major
  const int64_t i0 = items * blockIdx.x / gridDim.x, i1 = items * (blockIdx.x + 1) / gridDim.x;
  const size_t xbytes = size_t(kDiagChunk) * r_in * sizeof(double);
  const size_t dbytes = xbytes * r_out;
  double* sD = reinterpret_cast<double*>(dsm);
  unsigned char* sx = dsm + dbytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDiagStages; ++s) dmma::mbar_init(&full[s], 1);
    dmma::mbar_init(&dbar, 1);
    dmma::fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  auto issue = [&](int64_t it, int s) {
    const int64_t ib = it / p.M, m = it - ib * p.M;
    dmma::mbar_arrive_expect_tx(&full[s], uint32_t(xbytes));
    dmma::bulk_g2s(sx + size_t(s) * xbytes, p.in + (m * n_i + ib * kDiagChunk) * r_in, uint32_t(xbytes), &full[s]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < kDiagStages; ++s)
      if (i0 + s < i1) issue(i0 + s, s);
  const int r = threadIdx.x >> 1, h = threadIdx.x & 1;
  uint32_t phase = 0, dphase = 0;
  int s = 0;
  int64_t dblk = -1;
  for (int64_t it = i0; it < i1; ++it) {
    const int64_t ib = it / p.M, m = it - ib * p.M;
    if (ib != dblk) {                       // this range's next ii block: its D rows to smem
      __syncthreads();                      // everyone is done with the previous block
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        dmma::mbar_arrive_expect_tx(&dbar, uint32_t(dbytes));
        dmma::bulk_g2s(sD, p.core + size_t(ib) * kDiagChunk * r_in * r_out, uint32_t(dbytes), &dbar);
      }
      dmma::mbar_wait(&dbar, dphase);
      dphase ^= 1u;
      dblk = ib;
    }
    dmma::mbar_wait(&full[s], phase);
    const double* xr = reinterpret_cast<const double*>(sx + size_t(s) * xbytes) + size_t(r) * r_in;
    const double* D = sD + size_t(r) * r_in * RO;
    double acc[RO];
#pragma unroll
    for (int b = 0; b < RO; ++b) acc[b] = 0.0;
#pragma unroll 8
    for (int a = h; a < r_in; a += 2) {
      const double xa = xr[a];
#pragma unroll
      for (int b = 0; b < RO; ++b) acc[b] = fma(xa, D[a * RO + b], acc[b]);
    }
#pragma unroll
    for (int b = 0; b < RO; ++b) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], 1);
    if (h == 0) {
      const int64_t ii = ib * kDiagChunk + r;
      const int64_t row = m + (((m >> p.log2_q) * (n_i - 1)) << p.log2_q) + (ii << p.log2_q);
#pragma unroll
      for (int b = 0; b < RO; ++b) {
        QTT_CHECK_OUT(p, p.out + row * RO + b, 1);
        p.out[row * RO + b] = acc[b];
      }
    }
    __syncthreads();                        // stage s consumed
    if (threadIdx.x == 0 && it + kDiagStages < i1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(it + kDiagStages, s);
    }
    if (++s == kDiagStages) {
      s = 0;
      phase ^= 1u;
    }
  }
}

}  // namespace

cudaError_t launch_diag(const LevelArgs& a, cudaStream_t st, int num_sms) {
  if (a.r_in > kDiagMaxRin || a.r_out > kDiagMaxRank) return cudaErrorInvalidValue;
  if (a.r_out > kDiagMaxROut) {   // lanes over the outputs
    int64_t blocks = (a.M * a.n_i + 7) / 8;
    const int64_t capo = int64_t(num_sms) * 16;
    if (blocks > capo) blocks = capo;
    if (blocks < 1) blocks = 1;
    cudaLaunchAttribute attro[1];
    attro[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attro[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t co = {};
    co.gridDim = dim3(unsigned(blocks));
    co.blockDim = dim3(256);
    co.stream = st;
    co.attrs = attro;
    co.numAttrs = 1;
    return cudaLaunchKernelEx(&co, diag_out_kernel, a);
  }
  static const bool no_stream = std::getenv("QTT_DIAG_NO_STREAM") != nullptr;   // diagnostic (A/B)
  const size_t xb = size_t(kDiagChunk) * a.r_in * sizeof(double);
  const size_t smem_s = xb * (a.r_out + kDiagStages);
  if (!no_stream && a.n_i >= kDiagChunk && a.r_out <= kDiagMaxROut && smem_s <= kDiagStreamSmem) {
    using DiagFn = void (*)(const LevelArgs);
    static const DiagFn fns[kDiagMaxROut] = {diag_stream_kernel<1>, diag_stream_kernel<2>, diag_stream_kernel<3>,
                                             diag_stream_kernel<4>, diag_stream_kernel<5>, diag_stream_kernel<6>,
                                             diag_stream_kernel<7>, diag_stream_kernel<8>};
    // the smem attribute is per device: set once for each device this process uses
    static bool attr_set[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      for (DiagFn f : fns) {
        const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f),
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDiagStreamSmem));
        if (e != cudaSuccess) return e;
      }
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
    const int64_t items = int64_t(a.n_i / kDiagChunk) * a.M;
    int64_t blocks = items < num_sms ? items : num_sms;
    if (blocks < 1) blocks = 1;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t cs = {};
    cs.gridDim = dim3(unsigned(blocks));
    cs.blockDim = dim3(256);
    cs.dynamicSmemBytes = smem_s;
    cs.stream = st;
    cs.attrs = attrs;
    cs.numAttrs = 1;
    return cudaLaunchKernelEx(&cs, fns[a.r_out - 1], a);
  }
  const bool lane_ii = a.M < 32;
  const int64_t warps = lane_ii ? a.M * ((a.n_i + 31) / 32) : (a.M + 31) / 32 * a.n_i;
  int64_t blocks = (warps + 7) / 8;
  const int64_t cap = int64_t(num_sms) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(blocks));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // 16-byte row loads need even r_in (every row then starts 16-byte aligned)
  if (lane_ii) {
    if (a.r_in % 2 == 0) return cudaLaunchKernelEx(&cfg, diag_kernel<true, true>, a);
    return cudaLaunchKernelEx(&cfg, diag_kernel<false, true>, a);
  }
  if (a.r_in % 2 == 0) return cudaLaunchKernelEx(&cfg, diag_kernel<true, false>, a);
  return cudaLaunchKernelEx(&cfg, diag_kernel<false, false>, a);
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
                                                       dmma_threads(NB), smem);
}

bool pdl_enabled() {
  static const bool on = std::getenv("QTT_NO_PDL") == nullptr;
  return on;
}

cudaError_t launch_level_dmma(const LevelArgs& a, cudaStream_t st) {
  KernelFn f = lookup(a.KB, a.NB);
  if (!f) return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(dmma_threads(a.NB));
  cfg.dynamicSmemBytes = a.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, f, a);
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
