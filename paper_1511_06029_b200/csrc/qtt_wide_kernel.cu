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
//   * producer warp: per k-chunk of 32, the A chunk (two 64 x 16 boxes of a
//     2-D TMA tensor map over A, cp.async.bulk.tensor with the 128-byte
//     swizzle, so the A fragment loads are bank-conflict free; rows past M are
//     zero-filled by the TMA unit) and the W chunk (one contiguous
//     cp.async.bulk of fragment-packed doubles, 8-32 KiB, L2-resident across
//     tiles) land in a 4-stage mbarrier ring;
//   * 4 x CG consumer warps accumulate over all k-chunks of a tile in
//     registers (DMMA m8n8k4, as in qtt_dmma_kernel.cuh) and store with the
//     row-separation epilogue of the stage (out row m + Q*(s*(2^L-1) + ii)).
//
// This unit also holds the kernels that share that epilogue (tile_store):
//   * instances by MODE flags: 1 host-copy hooks, 2 fused shard exchange
//     (scatter_store into peer buffers), 4 split-K partials;
//   * split_reduce_kernel: the fixed-order sum of split-K partials;
//   * small_dmma_kernel: warp-tile stages straight from L2;
//   * shard_reduce_kernel: a part's fixed-order sum of its P receive slots (§9).
#include "qtt_dmma_kernel.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

namespace qtt {
namespace wide {
namespace {

using dmma::bulk_g2s;
using dmma::dmma_884;
using dmma::fence_mbar_init;
using dmma::mbar_arrive;
using dmma::mbar_arrive_expect_tx;
using dmma::mbar_init;
using dmma::mbar_wait;
using dmma::pdl_wait;

// A chunk in smem: kWideKBC boxes of [64 rows][16 doubles] = 8 KiB each, 128-byte
// swizzled (16-byte granule c of row r stored at granule c ^ (r % 8)).
constexpr uint32_t kABoxBytes = uint32_t(kDmmaRowsPerSubtile) * 16 * 8;
constexpr uint32_t kAStageBytes = kWideKBC * kABoxBytes;   // 16384
__host__ __device__ constexpr uint32_t b_chunk_bytes(int NB) { return uint32_t(kWideKBC) * NB * 32 * 32; }
__host__ __device__ constexpr uint32_t stage_bytes(int NB) { return kAStageBytes + b_chunk_bytes(NB); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dmma::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(dmma::smem_u32(bar))
      : "memory");
}

// Accumulate one k-chunk (kWideKBC k16 blocks) into c: 16 rows x NBC n8-blocks.
// A fragments come from a swizzled box: lane (g, t0) needs doubles
// 4*t0 .. 4*t0+3 (16-byte granules 2*t0, 2*t0+1) of rows row0 and row0 + 8,
// both congruent to g mod 8.  Operands are loaded one granule (two k4 steps)
// at a time so that only half of the A and B fragments are live at once.
template <int NB, int NBC>
__device__ __forceinline__ void chunk_mma(double (&c)[NBC][4], const unsigned char* sA, int row0,
                                          const double2* sB, int nb0, int lane) {
  const int t0 = lane & 3, g = lane >> 2;
#pragma unroll
  for (int kb = 0; kb < kWideKBC; ++kb) {
    const unsigned char* p0 = sA + kb * kABoxBytes + row0 * 128;
    const unsigned char* p1 = p0 + 8 * 128;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int off = ((2 * t0 + half) ^ g) * 16;
      const double2 x = *reinterpret_cast<const double2*>(p0 + off);
      const double2 y = *reinterpret_cast<const double2*>(p1 + off);
      double2 b[NBC];
#pragma unroll
      for (int nb = 0; nb < NBC; ++nb) b[nb] = sB[((kb * NB + nb0 + nb) * 32 + lane) * 2 + half];
#pragma unroll
      for (int nb = 0; nb < NBC; ++nb) {
        dmma_884(c[nb][0], c[nb][1], x.x, b[nb].x);
        dmma_884(c[nb][2], c[nb][3], y.x, b[nb].x);
      }
#pragma unroll
      for (int nb = 0; nb < NBC; ++nb) {
        dmma_884(c[nb][0], c[nb][1], x.y, b[nb].y);
        dmma_884(c[nb][2], c[nb][3], y.y, b[nb].y);
      }
    }
  }
}

// Row-separation epilogue (Alg. 2 line 8 for all L levels): column n = ii*r_out + b
// of GEMM row m goes to out[(m + Q*(s*(n_i-1) + ii)) * r_out + b], s = m / Q.
__device__ __forceinline__ int mout_dim(const LevelArgs&) { return 0; }
__device__ __forceinline__ int mout_dim(const FusedStage& p) { return p.mout_dim; }
__device__ __forceinline__ int mout_log2n(const LevelArgs&) { return 0; }
__device__ __forceinline__ int mout_log2n(const FusedStage& p) { return p.log2n; }

template <int NBC, class P>
__device__ __forceinline__ void tile_store(const double (&c)[NBC][4], const P& p, int64_t m_first,
                                           int n_first, int lane) {
  const int g = lane >> 2, t0 = lane & 3;
  const int md = mout_dim(p);
  if (md) {
    // last stage of a fused grid apply (r_out = 1): output row o of RHS s goes
    // to the natural-order grid at s N + morton_natural(o mod N)
    const int log2n = mout_log2n(p);
    const int64_t nmask = (int64_t(1) << log2n) - 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t m = m_first + g + 8 * h;
      if (m >= p.M) continue;
      const int64_t rowbase = m + (((m >> p.log2_q) * (p.n_i - 1)) << p.log2_q);
#pragma unroll
      for (int nb = 0; nb < NBC; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n_first + nb * 8 + 2 * t0 + e;
          if (n >= p.nout) continue;
          const int64_t o = rowbase + (int64_t(n) << p.log2_q);
          double* dst = p.out + (o & ~nmask) + morton_natural(o & nmask, md, log2n / md);
          QTT_CHECK_OUT(p, dst, 1);
          *dst = c[nb][2 * h + e];
        }
    }
    return;
  }
  const int r_out = p.r_out;
  const bool vec = (r_out % 2) == 0;
  // (ii, b) of this lane's first column, then advanced by 8 columns per n-block
  const int n_lane = n_first + 2 * t0;
  const int ii_lane = n_lane / r_out;
  const int b_lane = n_lane - ii_lane * r_out;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t m = m_first + g + 8 * h;
    if (m >= p.M) continue;
    const int64_t rowbase = m + (((m >> p.log2_q) * (p.n_i - 1)) << p.log2_q);
    int ii = ii_lane, b = b_lane;
#pragma unroll
    for (int nb = 0; nb < NBC; ++nb) {
      const int n = n_lane + nb * 8;
      if (n < p.nout) {
        double* dst = p.out + (rowbase + (int64_t(ii) << p.log2_q)) * r_out + b;
        QTT_CHECK_OUT(p, dst, vec ? 2 : 1);
        if (vec) {
          *reinterpret_cast<double2*>(dst) = make_double2(c[nb][2 * h], c[nb][2 * h + 1]);
        } else {
          dst[0] = c[nb][2 * h];
          if (n + 1 < p.nout) {
            const bool wrap = (b + 1 == r_out);
            double* d1 = p.out + (rowbase + (int64_t(ii + wrap) << p.log2_q)) * r_out + (wrap ? 0 : b + 1);
            QTT_CHECK_OUT(p, d1, 1);
            *d1 = c[nb][2 * h + 1];
          }
        }
      }
      b += 8;
      while (b >= r_out) {
        b -= r_out;
        ++ii;
      }
    }
  }
}

// Fused-stage epilogue through shared memory (r_out divides 32, Q a multiple
// of 16): the 16 x 32 warp tile covers 32 / r_out whole ii blocks, and each
// block's output is ONE contiguous run of 16 r_out doubles (rows m0..m0+15 of
// one RHS, b fastest).  A warp writes its tile (or its split-K partial) into
// its smem slot `ws` (512 doubles) in run order; the tile then leaves as 8
// pieces of 32 16-byte stores, 512 contiguous bytes per warp instruction --
// instead of 8-byte scattered stores (r_out = 1: 16 instructions of 4 x 64-byte
// pieces each).
__device__ __forceinline__ void runs_write(const double (&c)[4][4], int r, double* ws, int lane) {
  const int g = lane >> 2, t0 = lane & 3;
  const int lr = __ffs(r) - 1;                      // r = 2^lr
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = nb * 8 + 2 * t0 + e, row = g + 8 * h;
        const int b = col & (r - 1);
        ws[((col - b) << 4) + (row << lr) + b] = c[nb][2 * h + e];
      }
}

// The wide stage's plain epilogue with host-computed column offsets
// (LevelArgs::col_off): out + rowbase(m) r_out + col_off[n] -- one L1-cached
// load per column pair and one 64-bit multiply per row instead of the
// generic column walk (tile_store), so the epilogue the tile's warps run
// together is short (it is DMMA-idle time).
template <int NBC>
__device__ __forceinline__ void tile_store_cols(const double (&c)[NBC][4], const LevelArgs& p, int64_t m_first,
                                                int n_first, int lane) {
  const int g = lane >> 2, t0 = lane & 3;
  const bool vec = (p.r_out & 1) == 0;
  int64_t co[NBC];
#pragma unroll
  for (int nb = 0; nb < NBC; ++nb) {
    const int n = n_first + nb * 8 + 2 * t0;
    co[nb] = n < p.nout ? __ldg(p.col_off + n) : int64_t(-1);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t m = m_first + g + 8 * h;
    if (m >= p.M) continue;
    double* rowp = p.out + (m + (((m >> p.log2_q) * (p.n_i - 1)) << p.log2_q)) * p.r_out;
#pragma unroll
    for (int nb = 0; nb < NBC; ++nb) {
      if (co[nb] < 0) continue;
      double* dst = rowp + co[nb];
      QTT_CHECK_OUT(p, dst, vec ? 2 : 1);
      if (vec) {
        *reinterpret_cast<double2*>(dst) = make_double2(c[nb][2 * h], c[nb][2 * h + 1]);
      } else {
        dst[0] = c[nb][2 * h];
        const int n1 = n_first + nb * 8 + 2 * t0 + 1;   // odd r_out: the pair may wrap to the next ii
        if (n1 < p.nout) {
          const int64_t c1 = __ldg(p.col_off + n1);
          QTT_CHECK_OUT(p, rowp + c1, 1);
          rowp[c1] = c[nb][2 * h + 1];
        }
      }
    }
  }
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Fused shard exchange (r_out = 1): column n of GEMM row m goes to peers[n][m].
// A lane holds rows (g, g + 8) x columns (n, n + 1); one shuffle with the lane
// of the neighbouring row (g ^ 1) gives each lane two consecutive rows of ONE
// column, stored as one 16-byte peer store (NVLink: half the transactions of
// 8-byte stores).  M and the part's slot offset are even, so the pair never
// straddles the end of a slot.
template <int NBC>
__device__ __forceinline__ void scatter_store(const double (&c)[NBC][4], const LevelArgs& p, int64_t m_first,
                                              int n_first, int lane) {
  const int g = lane >> 2, t0 = lane & 3;
  const bool odd = g & 1;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t m_even = m_first + (g & ~1) + 8 * h;
#pragma unroll
    for (int nb = 0; nb < NBC; ++nb) {
      const double v0 = c[nb][2 * h], v1 = c[nb][2 * h + 1];   // (row g, col n), (row g, col n + 1)
      const double recv = __shfl_xor_sync(0xffffffffu, odd ? v0 : v1, 4);
      const int n = n_first + nb * 8 + 2 * t0 + (odd ? 1 : 0);
      if (m_even < p.M && n < p.nout) {
        double* dst = p.peers[n] + p.peer_offset + m_even;
        *reinterpret_cast<double2*>(dst) = odd ? make_double2(recv, v1) : make_double2(v0, recv);
      }
    }
  }
}

// Split-K (MODE & 4).  Tile t = tile_out * S + ks covers k-chunks
// [ks * kcps, min(nchunks, (ks + 1) * kcps)); each consumer warp stores its
// 16 x 8*NBC partial to slot (tile_out, ks, warp) of p.partial (lane-minor,
// 256 bytes per store instruction).  split_reduce_kernel, the next launch on
// the stream, sums the S slots in the fixed order ks = 0..S-1 (bitwise
// reproducible) and runs the ordinary row-separation epilogue.  (An in-kernel
// "last arrival reduces" protocol with per-tile counters read stale partials
// in ~1 of 150 applies of a K = 24320 stage even with gpu-scope fences on
// every lane and strong loads/stores; the kernel boundary is the one
// synchronisation that held.)
template <int NBC>
__device__ __forceinline__ void split_store(const double (&c)[NBC][4], const LevelArgs& p, int64_t tile_out, int ks,
                                            int warp, int cw, int slot, int lane) {
  double* mine = p.partial + ((tile_out * p.ksplit + ks) * cw + warp) * int64_t(slot);
#pragma unroll
  for (int nb = 0; nb < NBC; ++nb)
#pragma unroll
    for (int v = 0; v < 4; ++v) __stcg(mine + (nb * 4 + v) * 32 + lane, c[nb][v]);
}

template <int NB, int NBC, int MODE>
__device__ __forceinline__ void consumer(const LevelArgs& p, uint64_t* full, uint64_t* empty, const int64_t* tile_id,
                                         unsigned char* ring, int rg, int nb0, int lane, int warp = 0, int cw = 0,
                                         int slot = 0) {
  const int g = lane >> 2;
  double c[NBC][4];
  int chunk = 0;
  int tile_nch = p.nchunks;

  for (int it = 0;; ++it) {
    const int s = it % kWideStages;
    const uint32_t ph = uint32_t(it / kWideStages) & 1u;
    mbar_wait(&full[s], ph);
    const int64_t t = tile_id[s];
    if (t < 0) break;
    if (chunk == 0) {
#pragma unroll
      for (int nb = 0; nb < NBC; ++nb) c[nb][0] = c[nb][1] = c[nb][2] = c[nb][3] = 0.0;
      if (MODE & 4) {
        const int ks = int(t % p.ksplit);
        tile_nch = min(p.kcps, p.nchunks - ks * p.kcps);
      }
    }
    const unsigned char* st = ring + size_t(s) * stage_bytes(NB);
    chunk_mma<NB, NBC>(c, st, rg * 16 + g, reinterpret_cast<const double2*>(st + kAStageBytes), nb0, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++chunk == tile_nch) {
      chunk = 0;
      int64_t to = t;
      if (MODE & 4) {   // partial only; split_reduce_kernel stores the tile
        to = t / p.ksplit;
        split_store<NBC>(c, p, to, int(t - to * p.ksplit), warp, cw, slot, lane);
        continue;
      }
      int64_t rt;
      int cb;
      if (!(MODE & 2) && p.col_off) {   // tile < 2^31: multiply-shift instead of a 64-bit divide
        const uint32_t t32 = uint32_t(to);
        const uint32_t q = p.ncb_mul ? (__umulhi(t32, p.ncb_mul) >> p.ncb_shr) : (t32 >> p.ncb_shr);
        rt = q;
        cb = int(t32 - q * uint32_t(p.ncb));
      } else {
        rt = to / p.ncb;
        cb = int(to - rt * p.ncb);
      }
      if (MODE & 2) scatter_store<NBC>(c, p, rt * kDmmaRowsPerSubtile + rg * 16, (cb * NB + nb0) * 8, lane);
      else if (p.col_off) tile_store_cols<NBC>(c, p, rt * kDmmaRowsPerSubtile + rg * 16, (cb * NB + nb0) * 8, lane);
      else tile_store<NBC>(c, p, rt * kDmmaRowsPerSubtile + rg * 16, (cb * NB + nb0) * 8, lane);
      if ((MODE & 1) && p.done) {   // publish this warp's part of the tile to the D2H copy stream
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.done + (rt * kDmmaRowsPerSubtile) / p.done_rows, 1u);
      }
    }
  }
}

// MODE flags: 1 host-copy hooks (qtt_apply_host), 2 fused shard exchange, 4 split-K;
// instances 0, 1, 2, 4, 5
template <int NB, int MODE>
__global__ void __launch_bounds__(wide_threads(NB), NB <= 8 ? QTT_WIDE_CTAS : 1)
wide_dmma_kernel(const LevelArgs p, const __grid_constant__ CUtensorMap tmA) {
  constexpr int CG = wide_col_groups(NB);
  constexpr int CW = kDmmaRowGroups * CG;
  constexpr int NBW = (NB + CG - 1) / CG;
  constexpr int NB_1 = (NB - NBW) < NBW ? (NB - NBW) : NBW;
  constexpr int NB_2 = NB - NBW - NB_1;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  int64_t* tile_id = reinterpret_cast<int64_t*>(empty + kMaxStages);
  // the 128-byte swizzle needs 1024-byte aligned boxes
#ifdef QTT_WIDE_GENERIC_RING
  unsigned char* ring = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem) + kBarBytes + 1023) & ~uintptr_t(1023));
#else
  // as an offset from the shared array, so the operand loads stay LDS (an
  // integer round trip of the pointer made them generic LD.E.128, with
  // 64-bit addresses and a spill in the NB = 16 instance)
  const uint32_t smem_base = dmma::smem_u32(smem);
  unsigned char* ring = smem + (((smem_base + kBarBytes + 1023u) & ~1023u) - smem_base);
#endif

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWideStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  pdl_wait();
  __syncthreads();

  if (warp == CW) {
    // ---------------- producer warp (one elected lane): tile scheduler + TMA loads ----------------
    if (lane == 0) {
      const int64_t M = p.M;
      const int64_t ntiles = ((M + kDmmaRowsPerSubtile - 1) / kDmmaRowsPerSubtile) * p.ncb * ((MODE & 4) ? p.ksplit : 1);
      const uint32_t bbytes = b_chunk_bytes(NB);
      int it = 0;
      bool first = true;
      for (;;) {
        // the first tile is the CTA's own index (grid <= tiles): no L2 atomic in front of the first load
        const int64_t t = first ? int64_t(blockIdx.x) : int64_t(gridDim.x) + atomicAdd(p.tile_counter, 1);
        first = false;
        if (t >= ntiles) {
          const int s = it % kWideStages;
          mbar_wait(&empty[s], (uint32_t(it / kWideStages) & 1u) ^ 1u);
          tile_id[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        int64_t to = t;
        int ch0 = 0, ch1 = p.nchunks;
        if (MODE & 4) {   // split-K: consecutive tiles are the k-ranges of one output tile
          to = t / p.ksplit;
          ch0 = int(t - to * p.ksplit) * p.kcps;
          ch1 = min(p.nchunks, ch0 + p.kcps);
        }
        const int64_t rt = to / p.ncb;
        const int cb = int(to - rt * p.ncb);
        const int m0 = int(rt * kDmmaRowsPerSubtile);
        const double* bsrc = p.bpack + size_t(cb) * p.nchunks * (bbytes / 8);
        if ((MODE & 1) && p.ready) {   // this tile's rows of A must have arrived from the host
          const unsigned* f = p.ready + m0 / p.ready_rows;
          while (int(ld_acquire_u32(f) - p.ready_val) < 0) __nanosleep(200);
          // the rows are read by the TMA unit (async proxy): order it after the acquire
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int ch = ch0; ch < ch1; ++ch, ++it) {
          const int s = it % kWideStages;
          mbar_wait(&empty[s], (uint32_t(it / kWideStages) & 1u) ^ 1u);
          unsigned char* st = ring + size_t(s) * stage_bytes(NB);
          tile_id[s] = t;
          mbar_arrive_expect_tx(&full[s], kAStageBytes + bbytes);
#pragma unroll
          for (int kb = 0; kb < kWideKBC; ++kb)
            tma_load_2d(st + kb * kABoxBytes, &tmA, ch * kWideBK + kb * 16, m0, &full[s]);
          bulk_g2s(st + kAStageBytes, bsrc + size_t(ch) * (bbytes / 8), bbytes, &full[s]);
        }
      }
    }
    return;
  }
  const int rg = warp % kDmmaRowGroups;
  const int cg = warp / kDmmaRowGroups;
  constexpr int SLOT = split_slot_doubles(NB);
  if constexpr (CG == 4) {
    static_assert(NB % 4 == 0, "4 column groups need NB % 4 == 0");
    consumer<NB, NB / 4, MODE>(p, full, empty, tile_id, ring, rg, cg * (NB / 4), lane, warp, CW, SLOT);
  } else if (cg == 0) {
    consumer<NB, NBW, MODE>(p, full, empty, tile_id, ring, rg, 0, lane, warp, CW, SLOT);
  } else if (cg == 1) {
    if constexpr (NB_1 > 0) consumer<NB, NB_1, MODE>(p, full, empty, tile_id, ring, rg, NBW, lane, warp, CW, SLOT);
  } else {
    if constexpr (NB_2 > 0)
      consumer<NB, NB_2, MODE>(p, full, empty, tile_id, ring, rg, NBW + NB_1, lane, warp, CW, SLOT);
  }
}

// Split-K reduction: one warp per (output tile, consumer-warp slot) of the
// split stage; sums the S partials in fixed order and stores like the stage's
// own epilogue (with the host-copy "done" publication when hooks are set).
template <int NB, int NBC>
__device__ __forceinline__ void split_reduce_one(const LevelArgs& p, int64_t to, int w, int rg, int nb0, int lane) {
  constexpr int CW = kDmmaRowGroups * wide_col_groups(NB);
  constexpr int SLOT = split_slot_doubles(NB);
  double c[NBC][4];
#pragma unroll
  for (int nb = 0; nb < NBC; ++nb) c[nb][0] = c[nb][1] = c[nb][2] = c[nb][3] = 0.0;
  for (int ks = 0; ks < p.ksplit; ++ks) {
    const double* src = p.partial + ((to * p.ksplit + ks) * CW + w) * int64_t(SLOT);
#pragma unroll
    for (int nb = 0; nb < NBC; ++nb)
#pragma unroll
      for (int v = 0; v < 4; ++v) c[nb][v] += __ldcs(src + (nb * 4 + v) * 32 + lane);
  }
  const int64_t rt = to / p.ncb;
  const int cb = int(to - rt * p.ncb);
  if (p.col_off) tile_store_cols<NBC>(c, p, rt * kDmmaRowsPerSubtile + rg * 16, (cb * NB + nb0) * 8, lane);
  else tile_store<NBC>(c, p, rt * kDmmaRowsPerSubtile + rg * 16, (cb * NB + nb0) * 8, lane);
  if (p.done) {
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(p.done + (rt * kDmmaRowsPerSubtile) / p.done_rows, 1u);
  }
}

template <int NB>
__global__ void __launch_bounds__(128) split_reduce_kernel(const LevelArgs p) {
  pdl_wait();
  constexpr int CG = wide_col_groups(NB);
  constexpr int CW = kDmmaRowGroups * CG;
  constexpr int NBW = (NB + CG - 1) / CG;
  constexpr int NB_1 = (NB - NBW) < NBW ? (NB - NBW) : NBW;
  constexpr int NB_2 = NB - NBW - NB_1;
  const int lane = threadIdx.x & 31;
  const int64_t wg = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
  const int64_t tiles = (p.M + kDmmaRowsPerSubtile - 1) / kDmmaRowsPerSubtile * p.ncb;
  if (wg >= tiles * CW) return;
  const int64_t to = wg / CW;
  const int w = int(wg - to * CW);
  const int rg = w % kDmmaRowGroups, cg = w / kDmmaRowGroups;
  if constexpr (CG == 4) {
    split_reduce_one<NB, NB / 4>(p, to, w, rg, cg * (NB / 4), lane);
  } else if (cg == 0) {
    split_reduce_one<NB, NBW>(p, to, w, rg, 0, lane);
  } else if (cg == 1) {
    if constexpr (NB_1 > 0) split_reduce_one<NB, NB_1>(p, to, w, rg, NBW, lane);
  } else {
    if constexpr (NB_2 > 0) split_reduce_one<NB, NB_2>(p, to, w, rg, NBW + NB_1, lane);
  }
}

// Small stages (latency-bound, L2-resident): one warp per 16 x 32 output block
// (rows m0.., columns cb*32..), no smem, no barriers, no TMA.  Per k-step of 8
// a lane loads one 16-byte A granule per row half (k = 8p + 2 t0 + {0, 1}: the
// same k permutation as the resident kernel, so two k4 MMAs per load) and its
// 4 n-blocks x 2 B values as two contiguous 32-byte pieces of the packed
// operand (pack_small: [cb][p][lane][s][nb], s = the k4 step within the 8).
// One 16 x 32 warp tile of a small stage.  COHERENT: the A rows were written
// earlier in the same kernel (the fused apply below), so they are read through
// L2 (ld.global.cg), never through the non-coherent/L1 path.
template <bool COHERENT, class P>
__device__ __forceinline__ void small_tile(const P& p, int64_t wt, int lane) {
  const int64_t mt = wt / p.ncb;
  const int cb = int(wt - mt * p.ncb);
  const int64_t m0 = mt * kSmallRows;
  const int g = lane >> 2, t0 = lane & 3;
  const int K = p.K;
  const bool ok0 = m0 + g < p.M, ok1 = m0 + g + 8 < p.M;
  const double* a0 = p.in + (m0 + g) * K + 2 * t0;
  const double* a1 = a0 + int64_t(8) * K;
  const double4* bp = reinterpret_cast<const double4*>(p.bpack) + (int64_t(cb) * p.nchunks * 32 + lane) * 2;
  double c[4][4];
#pragma unroll
  for (int nb = 0; nb < 4; ++nb) c[nb][0] = c[nb][1] = c[nb][2] = c[nb][3] = 0.0;
#pragma unroll 4
  for (int q = 0; q < p.nchunks; ++q) {
    const int k = q * kSmallK + 2 * t0;
    double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
    if (k + 1 < K) {
      if (COHERENT) {
        if (ok0) x = __ldcg(reinterpret_cast<const double2*>(a0 + q * kSmallK));
        if (ok1) y = __ldcg(reinterpret_cast<const double2*>(a1 + q * kSmallK));
      } else {
        if (ok0) x = __ldg(reinterpret_cast<const double2*>(a0 + q * kSmallK));
        if (ok1) y = __ldg(reinterpret_cast<const double2*>(a1 + q * kSmallK));
      }
    } else if (k < K) {
      if (ok0) x.x = COHERENT ? __ldcg(a0 + q * kSmallK) : __ldg(a0 + q * kSmallK);
      if (ok1) y.x = COHERENT ? __ldcg(a1 + q * kSmallK) : __ldg(a1 + q * kSmallK);
    }
    const double4 b0 = bp[int64_t(q) * 64], b1 = bp[int64_t(q) * 64 + 1];
    const double bs0[4] = {b0.x, b0.y, b0.z, b0.w}, bs1[4] = {b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      dmma_884(c[nb][0], c[nb][1], x.x, bs0[nb]);
      dmma_884(c[nb][2], c[nb][3], y.x, bs0[nb]);
    }
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      dmma_884(c[nb][0], c[nb][1], x.y, bs1[nb]);
      dmma_884(c[nb][2], c[nb][3], y.y, bs1[nb]);
    }
  }
  tile_store<4>(c, p, m0, cb * kSmallCols, lane);
}

__global__ void __launch_bounds__(kSmallWarps * 32) small_dmma_kernel(const LevelArgs p) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t wt = int64_t(blockIdx.x) * kSmallWarps + (threadIdx.x >> 5);
  if (wt / p.ncb * kSmallRows >= p.M) return;
  small_tile<false>(p, wt, lane);
}

// ---- the fused apply (variant kFused)
//
// Grid-wide barrier: all CTAs are co-resident (cooperative launch).  bar[0]
// counts arrivals monotonically within a launch: barrier b (1-based) is
// passed once it reaches b * gridDim.x.  Thread 0 arrives after the CTA
// barrier with a gpu-scope release (the CTA's stage output, ordered before it
// by bar.sync) and polls with acquire loads; the next stage reads the
// intermediate with ld.global.cg (L2, coherent).  At exit every CTA adds one
// more arrival and the last one resets the counter to 0 for the next launch
// (all CTAs have passed every barrier by then; the next launch is
// stream-ordered after this one).
// Poll until the counter reaches target.  Watchdog: the default launch is not
// cooperative, so a grid that the device cannot co-schedule
// (an SM-limited context) would spin forever -- after 30 s the kernel traps
// instead, and the apply returns a CUDA error (QTT_FUSED_COOP=1 or
// qtt_set_fused(h, 0) avoid it there).
__device__ __forceinline__ void grid_spin(const unsigned* bar, unsigned target) {
  unsigned n = 0;
  unsigned long long t0 = 0;
  while (int(ld_acquire_u32(bar) - target) < 0) {
    if ((++n & 1023u) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (!t0) t0 = t;
      else if (t - t0 > 30000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    grid_spin(bar, target);
  }
  __syncthreads();
}

// The same barrier split in two (thread 0 only; the caller brackets it with
// __syncthreads): arrive, then -- after work that needs nobody else's output
// -- wait.
__device__ __forceinline__ void grid_arrive(unsigned* bar) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void grid_wait(unsigned* bar, unsigned target) { grid_spin(bar, target); }

__device__ __forceinline__ void grid_exit(unsigned* bar, unsigned total) {
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    if (old == total - 1) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(bar), "r"(0u) : "memory");
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// the timer read after v is available (v is an input of the asm: the read
// waits on v's scoreboard, e.g. the last DMMA into an accumulator)
__device__ __forceinline__ unsigned long long globaltimer_after(double v) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "d"(v));
  return t;
}

// Partial product of one 16 x 32 warp tile over k-steps [q0, q1) (k-steps of
// 8).  B comes from shared memory: the CTA's block of the stage's super-core
// for this tile's 32 columns, fragment-ordered [q][s][h][lane][2] (pack_fused)
// so each of the four 16-byte reads per k-step is conflict-free.  A comes
// straight from L2, software-pipelined: the next four k-steps' A fragments
// are in flight while the current four k-steps' 64 DMMAs run.  COHERENT: the
// A rows were written earlier in this launch -- read through L2
// (ld.global.cg).  K is even (K = n_i r_in, n_i >= 2), so a lane's k-pair is
// wholly inside K or wholly past it.
#ifndef QTT_FUSED_G
#define QTT_FUSED_G 4
#endif
constexpr int kFusedG = QTT_FUSED_G;   // k-steps of A in flight per group (build knob for A/B)
struct FusedA {
  double2 x[kFusedG], y[kFusedG];
};

// MORTON (fused grid apply, stage 0): a0 / a1 are QTT-order offsets of the
// lane's two rows from p.in, which holds the natural-order grid; each 16-byte
// load takes QTT indices 2t, 2t + 1 (x0 = 0, 1): two adjacent grid points.
template <bool COHERENT, bool MORTON = false>
__device__ __forceinline__ void fused_load_a(FusedA& o, const double* a0, const double* a1, int q, int q1, int K,
                                             int t0, bool ok0, bool ok1, const FusedStage& p) {
#pragma unroll
  for (int j = 0; j < kFusedG; ++j) {
    const int qq = q + j;
    const bool vk = qq < q1 && (qq * kSmallK + 2 * t0 < K);
    o.x[j] = make_double2(0.0, 0.0);
    o.y[j] = make_double2(0.0, 0.0);
    const double* e0 = a0 + qq * kSmallK;
    const double* e1 = a1 + qq * kSmallK;
    if (MORTON) {
      const int64_t nmask = (int64_t(1) << p.log2n) - 1, lv = p.log2n / p.in_dim;
      const int64_t i0 = e0 - p.in, i1 = e1 - p.in;
      e0 = p.in + ((i0 & ~nmask) + morton_natural(i0 & nmask, p.in_dim, int(lv)));
      e1 = p.in + ((i1 & ~nmask) + morton_natural(i1 & nmask, p.in_dim, int(lv)));
    }
    const double2* pa0 = reinterpret_cast<const double2*>(e0);
    const double2* pa1 = reinterpret_cast<const double2*>(e1);
    if (vk && ok0) o.x[j] = COHERENT ? __ldcg(pa0) : __ldg(pa0);
    if (vk && ok1) o.y[j] = COHERENT ? __ldcg(pa1) : __ldg(pa1);
  }
}

__device__ __forceinline__ void fused_mma(const FusedA& o, const double2* sB, int q, int q1, int lane,
                                          double (&c)[4][4]) {
#pragma unroll
  for (int j = 0; j < kFusedG; ++j) {
    const int qq = q + j;
    if (qq >= q1) break;
    const double2* b = sB + size_t(qq) * 128 + lane;      // [q][s][h][lane]
    const double2 b00 = b[0], b01 = b[32], b10 = b[64], b11 = b[96];
    const double bs0[4] = {b00.x, b00.y, b01.x, b01.y}, bs1[4] = {b10.x, b10.y, b11.x, b11.y};
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      dmma_884(c[nb][0], c[nb][1], o.x[j].x, bs0[nb]);
      dmma_884(c[nb][2], c[nb][3], o.y[j].x, bs0[nb]);
    }
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      dmma_884(c[nb][0], c[nb][1], o.x[j].y, bs1[nb]);
      dmma_884(c[nb][2], c[nb][3], o.y[j].y, bs1[nb]);
    }
  }
}

// One stage of the fused apply.  A unit of work is one 32-column block cb of
// the stage's output and kFusedWarps / ks row tiles of 16 rows: the CTA
// copies the super-core block of cb (K x 32 doubles) into shared memory with
// one bulk copy, and its warps take the row tiles, ks warps per tile, each
// over a contiguous 1/ks of the k-steps; the ks partial tiles meet in shared
// memory and the first warp of each tile adds them in the fixed order
// 0..ks-1 (deterministic; ks is fixed per plan, so results do not depend on
// nrhs) and runs the row-separation epilogue.  Units go to the CTAs
// round-robin, consecutive units sharing cb (its block stays hot in L2).
// Work units of a fused stage: (32-column block, group of row tiles), all
// counts precomputed on the host (FusedStage): the kernel multiplies and
// shifts, it never divides (an integer division is ~20-70 instructions, and
// at c1's size the stage is instruction-latency bound).
__device__ __forceinline__ int fused_cb(const FusedStage& p, int u) {      // u / rgroups
  return p.rg_mul ? int(__umulhi(uint32_t(u), p.rg_mul) >> p.rg_shr) : (u >> p.rg_shr);
}

// Thread 0: bulk-copy column block cb's super-core block into sB.
__device__ __forceinline__ void fused_issue_b(const FusedStage& p, int cb, double2* sB, uint64_t* bar) {
  const uint32_t bbytes = uint32_t(p.nchunks) * 128u * 16u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // sB's generic reads before the async write
  dmma::mbar_arrive_expect_tx(bar, bbytes);
  dmma::bulk_g2s(sB, p.bpack + size_t(cb) * p.nchunks * 256, bbytes, bar);
}

// Run-wise epilogue pieces with the tile's row base precomputed: piece k
// (double2 k * 32 + lane of the run-ordered tile) goes to out at run ii.
__device__ __forceinline__ void runs_store_piece_rb(const FusedStage& p, int64_t rowbase, int ii0, int k, int lane,
                                                    double2 v) {
  const int lr = p.lr, lrun = lr + 4;
  const int e2 = (k * 32 + lane) * 2;
  const int ii = ii0 + (e2 >> lrun);
  if (ii < p.n_i) {
    int64_t o = ((rowbase + (int64_t(ii) << p.log2_q)) << lr) + (e2 & ((1 << lrun) - 1));
    if (p.mout_dim) {   // fused grid apply (r_out = 1): QTT index o -> its natural-order grid point
      const int64_t nmask = (int64_t(1) << p.log2n) - 1;
      o = (o & ~nmask) + morton_natural(o & nmask, p.mout_dim, p.log2n / p.mout_dim);
    }
    double* dst = p.out + o;
    QTT_CHECK_OUT(p, dst, 2);
    *reinterpret_cast<double2*>(dst) = v;
  }
}

// One stage of the fused apply.  A unit of work is one 32-column block cb of
// the stage's output and kFusedWarps / KS row tiles of 16 rows: the CTA
// copies the super-core block of cb (K x 32 doubles) into shared memory with
// one bulk copy, and its warps take the row tiles, KS warps per tile, each
// over a contiguous 1/KS of the k-steps; the KS partial tiles meet in shared
// memory and are added in the fixed order 0..KS-1 (deterministic; KS is
// fixed per plan, so results do not depend on nrhs) before the
// row-separation epilogue.  Units go to the CTAs round-robin, consecutive
// units sharing cb (its block stays hot in L2).
template <bool COHERENT, bool PROF, bool MORTON = false>
__device__ __forceinline__ void fused_stage(const FusedStage& p, double* red, double2* sB, uint64_t* bar,
                                            uint32_t& nwait, bool prefetched, int lane,
                                            unsigned long long* dprof = nullptr,
                                            unsigned long long* wprof = nullptr) {
  const int lks = p.lks, KS = 1 << lks;              // warps per tile (power of two)
  const int lslots = 3 - lks;                         // log2(kFusedWarps / KS)
  const int w = threadIdx.x >> 5;
  const int slot = w >> lks, kp = w & (KS - 1);
  const int q0 = min(p.nchunks, kp * p.cps), q1 = min(p.nchunks, q0 + p.cps);
  const int t0 = lane & 3, g = lane >> 2;
  for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
    const int cb = fused_cb(p, u);
    const int mt = ((u - cb * p.rgroups) << lslots) + slot;
    const bool live = mt < p.mtiles;
    const int64_t m0 = int64_t(mt) * kSmallRows;
    const bool first = u == int(blockIdx.x);
    if (!first) __syncthreads();           // the previous unit is done with sB and red
    const bool rec = PROF && dprof && threadIdx.x == 0 && first;
    if (rec) dprof[0] = globaltimer();
    if (threadIdx.x == 0 && !(first && prefetched)) fused_issue_b(p, cb, sB, bar);
    // A fragments of the first k-steps while the super-core block lands
    const bool ok0 = live && m0 + g < p.M, ok1 = live && m0 + g + 8 < p.M;
    const double* a0 = p.in + (m0 + g) * p.K + 2 * t0;
    const double* a1 = a0 + int64_t(8) * p.K;
    FusedA fa, fb;
    if (q0 < q1) fused_load_a<COHERENT, MORTON>(fa, a0, a1, q0, q1, p.K, t0, ok0, ok1, p);
    double c[4][4];
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) c[nb][0] = c[nb][1] = c[nb][2] = c[nb][3] = 0.0;
    dmma::mbar_wait(bar, nwait & 1u);
    ++nwait;
    if (rec) dprof[1] = globaltimer();
    unsigned long long* wp = (PROF && wprof && first) ? wprof + w * 4 : nullptr;   // per-warp stamps (lane 0)
    if (wp && lane == 0) wp[0] = globaltimer_after(fa.x[0].x);
    if (live) {
      for (int q = q0; q < q1; q += 2 * kFusedG) {
        if (q + kFusedG < q1) fused_load_a<COHERENT, MORTON>(fb, a0, a1, q + kFusedG, q1, p.K, t0, ok0, ok1, p);
        fused_mma(fa, sB, q, q1, lane, c);
        if (q + kFusedG >= q1) break;
        if (q + 2 * kFusedG < q1) fused_load_a<COHERENT, MORTON>(fa, a0, a1, q + 2 * kFusedG, q1, p.K, t0, ok0, ok1, p);
        fused_mma(fb, sB, q + kFusedG, q1, lane, c);
      }
    }
    if (rec) dprof[2] = globaltimer_after(c[0][0]);
    if (wp && lane == 0) wp[1] = globaltimer_after(c[3][3] + c[0][0]);
    double* wslot = red + size_t(w) * 16 * 32;     // this warp's own partial slot
    if (p.runs) {
      // run-wise epilogue: every row of the tile in one RHS (Q % 16 == 0), r_out | 32
      const int64_t rowbase = m0 + (((m0 >> p.log2_q) * (p.n_i - 1)) << p.log2_q);
      const int ii0 = (cb * kSmallCols) >> p.lr;
      runs_write(c, p.r_out, wslot, lane);
      if (KS == 1) {
        __syncwarp();
        if (live) {
          const double2* ws2 = reinterpret_cast<const double2*>(wslot);
#pragma unroll
          for (int k = 0; k < 8; ++k) runs_store_piece_rb(p, rowbase, ii0, k, lane, ws2[k * 32 + lane]);
        }
        __syncwarp();
      } else {
        // split-K: every warp of the tile wrote its partial in run order; the
        // tile's KS warps each reduce and store 8 / KS of its 8 pieces (sum in
        // the fixed order 0..KS-1: the same values, bitwise, as one warp
        // adding the partials in that order)
        __syncthreads();
        if (wp && lane == 0) wp[2] = globaltimer();
        if (live) {
          const double2* base = reinterpret_cast<const double2*>(red + size_t(slot) * KS * 16 * 32);
          for (int k = kp; k < 8; k += KS) {
            double2 acc = base[k * 32 + lane];
            for (int j = 1; j < KS; ++j) {
              const double2 o = base[j * 256 + k * 32 + lane];
              acc.x += o.x;
              acc.y += o.y;
            }
            runs_store_piece_rb(p, rowbase, ii0, k, lane, acc);
          }
        }
      }
      if (rec) dprof[3] = globaltimer();
      if (wp && lane == 0) wp[3] = globaltimer();
      continue;
    }
    if (KS == 1) {
      if (live) tile_store<4>(c, p, m0, cb * kSmallCols, lane);
      if (rec) dprof[3] = globaltimer();
      if (wp && lane == 0) wp[3] = globaltimer();
      continue;
    }
    // partials [warp][value][lane]: every access is 32 consecutive doubles (no bank conflicts)
    double* mine = red + size_t(w) * 16 * 32 + lane;
    if (kp) {
#pragma unroll
      for (int nb = 0; nb < 4; ++nb)
#pragma unroll
        for (int v = 0; v < 4; ++v) mine[(nb * 4 + v) * 32] = c[nb][v];
    }
    __syncthreads();
    if (wp && lane == 0) wp[2] = globaltimer();
    if (kp == 0 && live) {
      for (int j = 1; j < KS; ++j) {
        const double* o = red + size_t(w + j) * 16 * 32 + lane;
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int v = 0; v < 4; ++v) c[nb][v] += o[(nb * 4 + v) * 32];
      }
      if (wp && lane == 0) wp[2] = globaltimer_after(c[3][3] + c[0][0]);   // reduced
      tile_store<4>(c, p, m0, cb * kSmallCols, lane);
      if (rec) dprof[3] = globaltimer();
      if (wp && lane == 0) wp[3] = globaltimer();
    }
  }
}

// The whole apply of a latency-bound problem in ONE persistent launch: the
// plan's stages one after another, each spread over every warp of the grid
// (fused_stage), separated by grid barriers instead of kernel boundaries; the
// intermediates (two ping-pong buffers) stay in L2.
// PROF: the diagnostic instance (QTT_FUSED_PROFILE) with %globaltimer stamps;
// the production instance carries no profiling code.
template <bool PROF, bool MORTON>
__global__ void __launch_bounds__(kFusedWarps * 32) fused_small_kernel(const __grid_constant__ FusedArgs a) {
  __shared__ __align__(16) double red[kFusedWarps * 32 * 16];   // split-K partials, 32 KiB
  __shared__ __align__(8) uint64_t bar;
  extern __shared__ __align__(128) unsigned char fsm[];          // the super-core block of a unit
  double2* sB = reinterpret_cast<double2*>(fsm);
  if (threadIdx.x == 0) {
    dmma::mbar_init(&bar, 1);
    dmma::fence_mbar_init();
  }
  __syncthreads();
  // the first stage's super-core block is static (written at qtt_create, never
  // by a kernel): its copy starts before griddepcontrol.wait, overlapping the
  // previous kernel on the stream
  const bool prefetch0 = int(blockIdx.x) < a.st[0].units;
  if (threadIdx.x == 0 && prefetch0) fused_issue_b(a.st[0], fused_cb(a.st[0], blockIdx.x), sB, &bar);
  pdl_wait();
  unsigned long long* prof = (PROF && a.prof) ? a.prof + size_t(blockIdx.x) * kFusedProfSlots : nullptr;
  if (prof && threadIdx.x == 0) prof[0] = globaltimer();
  const int lane = threadIdx.x & 31;
  uint32_t nwait = 0;
  unsigned nbar = 0;
  bool prefetched = prefetch0;
  if (a.pre_dim) {   // Morton gather of the grid into QTT order (fused grid apply)
    const int64_t nmask = (int64_t(1) << a.pre_log2n) - 1;
    const int lv = a.pre_log2n / a.pre_dim;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < a.pre_total;
         e += int64_t(gridDim.x) * blockDim.x)
      a.pre_dst[e] = __ldg(a.pre_src + (e & ~nmask) + morton_natural(e & nmask, a.pre_dim, lv));
    grid_barrier(a.bar, ++nbar * gridDim.x);
  }
  for (int s = 0; s < a.nstages; ++s) {
    // the last stage: let the next kernel on the stream launch onto the SMs
    // this grid leaves free (it only stages its static super-core block before
    // its own griddepcontrol.wait, which waits for this grid to complete)
    if (s + 1 == a.nstages && a.early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int rep = 0; rep < a.repeat; ++rep) {
      if (prof && rep + 1 == a.repeat && rep > 0) {
        __syncthreads();
        if (threadIdx.x == 0) prof[2 * s] = globaltimer();   // timing of the last repeat only
      }
      unsigned long long* dp = prof ? prof + 2 * kFusedMaxStages + 2 + 4 * s : nullptr;
      unsigned long long* wpp = prof ? prof + kFusedProfBase + s * kFusedWarps * 4 : nullptr;
      if (MORTON && s == 0)           // the natural-order grid, gathered by the A loads (own instance)
        fused_stage<false, PROF, true>(a.st[s], red, sB, &bar, nwait, prefetched, lane, dp, wpp);
      else if (s == 0 && !a.pre_dim)  // x itself: written before this launch, read-only path
        fused_stage<false, PROF>(a.st[s], red, sB, &bar, nwait, prefetched, lane, dp, wpp);
      else                        // written earlier in this launch: through L2
        fused_stage<true, PROF>(a.st[s], red, sB, &bar, nwait, prefetched, lane, dp, wpp);
      prefetched = false;
      if (rep + 1 < a.repeat) grid_barrier(a.bar, ++nbar * gridDim.x);
    }
    if (prof) {
      __syncthreads();
      if (threadIdx.x == 0) prof[1 + 2 * s] = globaltimer();
    }
    if (s + 1 < a.nstages) {
      // split barrier: arrive, start the copy of the next stage's first
      // super-core block (static data, needs nobody's output), then wait
      __syncthreads();
      if (threadIdx.x == 0) {
        grid_arrive(a.bar);
        const FusedStage& nx = a.st[s + 1];
        if (int(blockIdx.x) < nx.units) fused_issue_b(nx, fused_cb(nx, blockIdx.x), sB, &bar);
        grid_wait(a.bar, ++nbar * gridDim.x);
      } else {
        ++nbar;
      }
      prefetched = int(blockIdx.x) < a.st[s + 1].units;
      __syncthreads();
    }
    if (prof && threadIdx.x == 0) prof[2 + 2 * s] = globaltimer();
  }
  grid_exit(a.bar, (nbar + 1) * gridDim.x);
}

using KernelFn = void (*)(const LevelArgs, const CUtensorMap);

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

template <int MODE>
KernelFn lookup_m(int NB) {
  switch (NB) {
    case 4: return &wide_dmma_kernel<4, MODE>;
    case 8: return &wide_dmma_kernel<8, MODE>;
    case 12: return &wide_dmma_kernel<12, MODE>;
    case 16: return &wide_dmma_kernel<16, MODE>;
    default: return nullptr;
  }
}

// mode flags: 1 host-copy pipelining (qtt_apply_host), 2 fused shard exchange,
// 4 split-K
KernelFn lookup(int NB, int mode) {
  switch (mode) {
    case 0: return lookup_m<0>(NB);
    case 1: return lookup_m<1>(NB);
    case 2: return lookup_m<2>(NB);
    case 4: return lookup_m<4>(NB);
    case 5: return lookup_m<5>(NB);
    default: return nullptr;
  }
}

__global__ void shard_reduce_kernel(const double2* __restrict__ recv, double2* __restrict__ y, int parts,
                                    int64_t count2) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count2; t += int64_t(gridDim.x) * blockDim.x) {
    double2 acc = recv[t];
    for (int g = 1; g < parts; ++g) {
      const double2 v = recv[int64_t(g) * count2 + t];
      acc.x += v.x;
      acc.y += v.y;
    }
    y[t] = acc;
  }
}

}  // namespace
}  // namespace wide

size_t wide_smem_bytes(int NB) { return kBarBytes + 1024 + size_t(kWideStages) * wide::stage_bytes(NB); }

cudaError_t wide_prepare(int NB, size_t smem) {
  for (int mode : {0, 1, 2, 4, 5}) {
    wide::KernelFn f = wide::lookup(NB, mode);
    if (!f) return cudaErrorInvalidValue;
    const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f),
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_wide(const LevelArgs& a, cudaStream_t st) {
  const bool split = a.ksplit > 1;
  if (split && (a.peers || !a.partial)) return cudaErrorInvalidValue;
  // the split kernel's tiles store partials only; the done hook belongs to the reduce launch
  LevelArgs am = a;
  if (split) am.done = nullptr;
  const bool hooks = am.ready != nullptr || am.done != nullptr;
  wide::KernelFn f = wide::lookup(a.NB, a.peers ? 2 : (split ? 4 : 0) | (hooks ? 1 : 0));
  auto encode = wide::encode_fn();
  if (!f || !encode) return cudaErrorInvalidValue;
  // A viewed as a 2-D tensor [M rows][K doubles], boxes of 64 rows x 16 doubles
  CUtensorMap map;
  const cuuint64_t dims[2] = {cuuint64_t(a.K), cuuint64_t(a.M)};
  const cuuint64_t strides[1] = {cuuint64_t(a.K) * sizeof(double)};
  const cuuint32_t box[2] = {16, cuuint32_t(kDmmaRowsPerSubtile)};
  const cuuint32_t estr[2] = {1, 1};
  if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(a.in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(wide_threads(a.NB));
  cfg.dynamicSmemBytes = a.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, f, am, map);
  if (e != cudaSuccess || !split) return e;
  // split-K: the fixed-order reduction + epilogue as the next launch
  const int64_t tiles = (a.M + kDmmaRowsPerSubtile - 1) / kDmmaRowsPerSubtile * a.ncb;
  const int64_t warps = tiles * wide_consumer_warps(a.NB);
  cudaLaunchConfig_t rc = cfg;
  rc.gridDim = dim3(unsigned((warps + 3) / 4));
  rc.blockDim = dim3(128);
  rc.dynamicSmemBytes = 0;
  switch (a.NB) {
    case 4: return cudaLaunchKernelEx(&rc, wide::split_reduce_kernel<4>, a);
    case 8: return cudaLaunchKernelEx(&rc, wide::split_reduce_kernel<8>, a);
    case 12: return cudaLaunchKernelEx(&rc, wide::split_reduce_kernel<12>, a);
    case 16: return cudaLaunchKernelEx(&rc, wide::split_reduce_kernel<16>, a);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_small(const LevelArgs& a, cudaStream_t st) {
  const int64_t wtiles = (a.M + kSmallRows - 1) / kSmallRows * a.ncb;
  const int64_t blocks = (wtiles + kSmallWarps - 1) / kSmallWarps;
  if (blocks > 0x7fffffff || (a.K % 2)) return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(blocks));
  cfg.blockDim = dim3(kSmallWarps * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, wide::small_dmma_kernel, a);
}

bool fused_cooperative() {
  static const bool coop = std::getenv("QTT_FUSED_COOP") != nullptr;
  return coop;
}

cudaError_t fused_prepare() {
  for (auto f : {wide::fused_small_kernel<false, false>, wide::fused_small_kernel<true, false>,
                 wide::fused_small_kernel<false, true>, wide::fused_small_kernel<true, true>}) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFusedMaxBBytes));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_fused(const FusedArgs& a, int grid, cudaStream_t st, bool pdl) {
  if (grid < 1 || a.nstages < 1 || a.nstages > kFusedMaxStages || a.smem > kFusedMaxBBytes)
    return cudaErrorInvalidValue;
  // Not a cooperative launch by default: a cooperative launch costs ~5 us more
  // host time and waits for the previous kernel to drain (no PDL overlap):
  // c1 12.3 vs 9.4 us per back-to-back apply.  Co-residency holds without it:
  // grid <= SMs at one CTA per SM (the kernel's registers fill an SM), and
  // the grid's own PDL dependents launch only after every CTA of this grid
  // ran its trigger.  QTT_FUSED_COOP=1 restores the cooperative attribute.
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = fused_cooperative() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl && pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(kFusedWarps * 32);
  cfg.dynamicSmemBytes = a.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (a.st[0].in_dim)   // fused grid apply gathering in stage 0: its own instance
    return a.prof ? cudaLaunchKernelEx(&cfg, wide::fused_small_kernel<true, true>, a)
                  : cudaLaunchKernelEx(&cfg, wide::fused_small_kernel<false, true>, a);
  return a.prof ? cudaLaunchKernelEx(&cfg, wide::fused_small_kernel<true, false>, a)
                : cudaLaunchKernelEx(&cfg, wide::fused_small_kernel<false, false>, a);
}

cudaError_t launch_shard_reduce(const double* recv, double* y, int parts, int64_t count, cudaStream_t st,
                                int num_sms) {
  if (count % 2) return cudaErrorInvalidValue;
  const int64_t c2 = count / 2;
  int64_t blocks = (c2 + 255) / 256;
  blocks = blocks > int64_t(num_sms) * 8 ? int64_t(num_sms) * 8 : (blocks < 1 ? 1 : blocks);
  wide::shard_reduce_kernel<<<int(blocks), 256, 0, st>>>(reinterpret_cast<const double2*>(recv),
                                                         reinterpret_cast<double2*>(y), parts, c2);
  return cudaGetLastError();
}

}  // namespace qtt
