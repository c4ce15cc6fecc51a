// Morton pack / unpack: natural grid order <-> QTT (hierarchical) order.
//
// the volume grid's N = 2^d points are indexed "according
// to successive bisection of the domain along each coordinate direction (i.e.,
// Morton ordered)"; Remark rem:interlace: the ordering defines the
// hierarchical partition the QTT ranks depend on.  Convention (R18,
// SPEC S:114): QTT index bit dim*l + a = bit l of coordinate a (a = 0 x, 1 y,
// 2 z), l = 0 the finest level; the natural grid is row-major with x fastest.
//
// Both directions are HBM-bound permutations (8 bytes read + 8 written per
// element).  Tiled path: one CTA moves one aligned block of 2^12 consecutive
// QTT indices = a 16^3 cube (dim 3) or 64^2 square (dim 2) of the grid,
// reading/writing the grid side in full 128-byte (dim 3) or 512-byte (dim 2)
// rows and the QTT side as one contiguous 32 KiB run, through an XOR-swizzled
// smem tile (bank-conflict free both ways), streaming loads/stores (.cs).
// Pack, whose scattered side is the read side, reads 256-byte (dim 3) grid
// rows: in 3-D a CTA moves the z_3 half of two x-adjacent tiles (32 x 16 x 8
// points, 32 KiB of static smem, two 16 KiB QTT runs; morton_pack3_half_kernel),
// in 2-D two x-adjacent tiles (64 KiB dynamic smem); consecutive CTAs take
// x-adjacent units.  Measured at 256^3: pack 5.2 TB/s = 80% of HBM (5.1 with two
// whole tiles per CTA, 70% with one tile and 128-byte rows), unpack 92%; one
// tile keeps static smem (a dynamic 32 KiB tile cost unpack 15%, from the
// carveout the driver picked).
// Grids smaller than one tile use a per-element kernel.
#include "qtt_internal.h"

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace qtt {
namespace {

constexpr int kTileBits = 12;                 // 4096 elements per CTA
constexpr int kTile = 1 << kTileBits;
constexpr int kThreads = 256;

// coordinate bits of a QTT index (de-interleave), dim in {1,2,3}
__device__ __forceinline__ void deinterleave(int64_t q, int dim, int levels, int64_t (&c)[3]) {
  c[0] = c[1] = c[2] = 0;
  for (int l = 0; l < levels; ++l)
    for (int a = 0; a < dim; ++a) c[a] |= ((q >> (dim * l + a)) & 1) << l;
}

// natural row-major offset of coordinates (x fastest)
__device__ __forceinline__ int64_t natural(const int64_t (&c)[3], int dim, int levels) {
  int64_t off = 0;
  for (int a = dim - 1; a >= 0; --a) off = (off << levels) | c[a];
  return off;
}

template <bool PACK>
__global__ void morton_simple_kernel(const double* __restrict__ in, double* __restrict__ out, int dim, int levels,
                                     int64_t total, int64_t N) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = t / N, q = t - s * N;
    int64_t c[3];
    deinterleave(q, dim, levels, c);
    const int64_t g = s * N + natural(c, dim, levels);
    if (PACK) out[t] = in[g];
    else out[g] = in[t];
  }
}

// Tile of 2^12 consecutive QTT indices.  dim 3: 16 x 16 x 16 (4 bits per axis),
// dim 2: 64 x 64 (6 bits per axis).  smem holds the tile in natural order,
// rows of R doubles, with x XOR-swizzled per row so that both access patterns
// are bank-conflict free for 8-byte elements (each half-warp touching 16
// distinct bank pairs): the grid side reads 16 consecutive x of one row; the
// QTT side reads 16 consecutive local indices u, i.e. x in c + {0..3} on 4
// rows that differ in (y_0, z_0) (dim 3) or (y_0, y_1) (dim 2) -- the swizzle
// puts those 4 rows on 4 different 4-aligned x offsets.
template <int DIM>
__device__ __forceinline__ int swz(int row) {
  if (DIM == 3) return 4 * ((row & 1) | (((row >> 4) & 1) << 1));   // row = z*16 + y: (y_0, z_0)
  return 4 * (row & 3);                                               // row = y: (y_0, y_1)
}

template <int DIM, bool PACK, int TX>
__global__ void __launch_bounds__(kThreads) morton_tile_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                               int levels, int64_t N) {
  constexpr int B = kTileBits / DIM;          // bits per axis inside the tile
  constexpr int R = 1 << B;                   // x extent of one tile
  constexpr int LT = TX == 2 ? 1 : 0;
  constexpr int RW = R * TX;                  // smem row length: TX x-adjacent tiles
  constexpr int ELEMS = kTile * TX;
  // one tile: static smem (lets the driver size the carveout for 7 CTAs/SM); two: dynamic
  __shared__ __align__(16) double tile_static[TX == 1 ? kTile : 2];
  extern __shared__ __align__(16) double tile_dyn[];
  double* tile = TX == 1 ? tile_static : tile_dyn;

  const int64_t units_per_rhs = (N >> kTileBits) >> LT;
  const int64_t s = blockIdx.x / units_per_rhs;
  const int64_t bid = blockIdx.x - s * units_per_rhs;
  // Consecutive CTAs take x-adjacent units (natural order of the tile grid), so
  // the CTAs resident together cover whole grid rows.  A unit is TX tiles
  // adjacent in x, i.e. consecutive in QTT order (x bit B is QTT bit kTileBits).
  const int tb = levels - B;                  // tile-coordinate bits per axis
  int64_t c0[3] = {0, 0, 0};
  {
    const int64_t xm = (int64_t(1) << (tb - LT)) - 1, m = (int64_t(1) << tb) - 1;
    c0[0] = (bid & xm) << (B + LT);
    const int64_t r = bid >> (tb - LT);
    c0[1] = (r & m) << B;
    if (DIM == 3) c0[2] = (r >> tb) << B;
  }
  int64_t tq = 0;                             // QTT index of the first tile
  for (int l = 0; l < tb; ++l)
    for (int a = 0; a < DIM; ++a) tq |= ((c0[a] >> (B + l)) & 1) << (DIM * l + a);
  const int64_t n = int64_t(1) << levels;
  const int64_t gbase = s * N + (DIM == 3 ? (c0[2] * n + c0[1]) * n + c0[0] : c0[1] * n + c0[0]);
  const int64_t qbase = s * N + (tq << kTileBits);

  // smem slot of local QTT index u (tile u >> kTileBits of the unit)
  auto slot_of_u = [](int u) {
    int x = (u >> kTileBits) * R, y = 0, z = 0;
#pragma unroll
    for (int l = 0; l < B; ++l) {
      x |= ((u >> (DIM * l)) & 1) << l;
      y |= ((u >> (DIM * l + 1)) & 1) << l;
      if (DIM == 3) z |= ((u >> (DIM * l + 2)) & 1) << l;
    }
    const int row = DIM == 3 ? z * R + y : y;
    return row * RW + (x ^ swz<DIM>(row));
  };
  // global offset (from gbase) and smem slot of the e-th element in natural order
  auto grid_of_e = [n](int e, int64_t& goff, int& slot) {
    const int x = e & (RW - 1), row = e >> (B + LT);   // row = z*R + y (dim 3) or y (dim 2)
    const int y = row & (R - 1), z = row >> B;
    goff = (DIM == 3 ? (int64_t(z) * n + y) * n : int64_t(y) * n) + x;
    slot = row * RW + (x ^ swz<DIM>(row));
  };

  // 16-byte accesses on both sides: x pairs (x even, x + 1) stay adjacent under
  // the swizzle (it flips only bits 2-3 of x), and u pairs are x pairs.
  double2* tile2 = reinterpret_cast<double2*>(tile);
  if (PACK) {
#pragma unroll
    for (int e = 2 * threadIdx.x; e < ELEMS; e += 2 * kThreads) {
      int64_t goff;
      int slot;
      grid_of_e(e, goff, slot);
      const double2* src = reinterpret_cast<const double2*>(in + gbase + goff);
      tile2[slot >> 1] = __ldcs(src);
    }
    __syncthreads();
#pragma unroll
    for (int u = 2 * threadIdx.x; u < ELEMS; u += 2 * kThreads)
      __stcs(reinterpret_cast<double2*>(out + qbase + u), tile2[slot_of_u(u) >> 1]);
  } else {
#pragma unroll
    for (int u = 2 * threadIdx.x; u < ELEMS; u += 2 * kThreads)
      tile2[slot_of_u(u) >> 1] = __ldcs(reinterpret_cast<const double2*>(in + qbase + u));
    __syncthreads();
#pragma unroll
    for (int e = 2 * threadIdx.x; e < ELEMS; e += 2 * kThreads) {
      int64_t goff;
      int slot;
      grid_of_e(e, goff, slot);
      __stcs(reinterpret_cast<double2*>(out + gbase + goff), tile2[slot >> 1]);
    }
  }
}

// 3-D pack, half-cube units: 32 (x) x 16 (y) x 8 (z) grid points = the z_3
// half of two x-adjacent 16^3 tiles.  The grid reads are 256-byte rows (as with
// two tiles per CTA), the QTT side is two contiguous 16 KiB runs (the half zh
// of QTT blocks tq and tq + 1), and the unit is 32 KiB of STATIC shared memory,
// so 7 CTAs fit an SM as in unpack (two whole tiles need 64 KiB: 3 CTAs).
__global__ void __launch_bounds__(kThreads) morton_pack3_half_kernel(const double* __restrict__ in,
                                                                     double* __restrict__ out, int levels,
                                                                     int64_t N) {
  constexpr int B = 4, R = 16, RW = 32;
  __shared__ __align__(16) double tile[kTile];
  const int64_t units_per_rhs = N >> kTileBits;            // (N / 4096 / 2 tile pairs) x 2 halves
  const int64_t s = blockIdx.x / units_per_rhs;
  const int64_t hb = blockIdx.x - s * units_per_rhs;
  // consecutive CTAs: x-adjacent tile pairs, then the two z halves, then y, z
  const int tb = levels - B;
  const int64_t xm = (int64_t(1) << (tb - 1)) - 1, m = (int64_t(1) << tb) - 1;
  const int64_t cx = (hb & xm) << (B + 1);
  const int64_t r0 = hb >> (tb - 1);
  const int zh = int(r0 & 1);
  const int64_t r = r0 >> 1;
  const int64_t cy = (r & m) << B, cz = (r >> tb) << B;
  int64_t tq = 0;                                          // QTT index of the first tile
  for (int l = 0; l < tb; ++l) {
    tq |= ((cx >> (B + l)) & 1) << (3 * l);
    tq |= ((cy >> (B + l)) & 1) << (3 * l + 1);
    tq |= ((cz >> (B + l)) & 1) << (3 * l + 2);
  }
  const int64_t n = int64_t(1) << levels;
  const int64_t gbase = s * N + ((cz + 8 * zh) * n + cy) * n + cx;
  const int64_t qbase = s * N + (tq << kTileBits) + (int64_t(zh) << (kTileBits - 1));
  double2* tile2 = reinterpret_cast<double2*>(tile);
#pragma unroll
  for (int e = 2 * threadIdx.x; e < kTile; e += 2 * kThreads) {
    const int x = e & (RW - 1), row = e >> 5;              // row = z * 16 + y, z in 0..7
    const int y = row & (R - 1), z = row >> B;
    const double2* src = reinterpret_cast<const double2*>(in + gbase + (int64_t(z) * n + y) * n + x);
    tile2[(row * RW + (x ^ swz<3>(row))) >> 1] = __ldcs(src);
  }
  __syncthreads();
#pragma unroll
  for (int u = 2 * threadIdx.x; u < kTile; u += 2 * kThreads) {
    const int t = u >> (kTileBits - 1), w = u & ((kTile >> 1) - 1);   // tile of the pair, index in its half
    int x = t * R, y = 0, z = 0;
#pragma unroll
    for (int l = 0; l < B; ++l) {
      x |= ((w >> (3 * l)) & 1) << l;
      y |= ((w >> (3 * l + 1)) & 1) << l;
      if (l < B - 1) z |= ((w >> (3 * l + 2)) & 1) << l;
    }
    const int row = z * R + y;
    __stcs(reinterpret_cast<double2*>(out + qbase + (int64_t(t) << kTileBits) + w),
           tile2[(row * RW + (x ^ swz<3>(row))) >> 1]);
  }
}

template <int DIM, bool PACK, int TX>
cudaError_t launch_tile(const double* in, double* out, int levels, int64_t N, int64_t nrhs, cudaStream_t st) {
  const int64_t blocks = nrhs * ((N >> kTileBits) / TX);
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  constexpr size_t smem = TX == 1 ? 0 : size_t(kTile) * TX * sizeof(double);
  auto f = morton_tile_kernel<DIM, PACK, TX>;
  if (smem > 48 * 1024) {
    const cudaError_t attr =   // per device; cheap
        cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (attr != cudaSuccess) return attr;
  }
  f<<<int(blocks), kThreads, smem, st>>>(in, out, levels, N);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_morton(const double* in, double* out, int dim, int levels, int64_t nrhs, bool pack,
                          cudaStream_t st, int num_sms) {
  const int d = dim * levels;
  const int64_t N = int64_t(1) << d;
  const bool aligned = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const bool tiled = aligned && ((dim == 3 && levels >= 4) || (dim == 2 && levels >= 6));
  if (tiled) {
    // pack reads the grid side: two x-adjacent tiles per CTA (256-byte rows)
    // where the grid has them (79% vs 70% of HBM at 256^3); unpack's scattered
    // side is the write side, which one tile per CTA already streams at 92%
    const bool two = levels >= (kTileBits / dim) + 1;
    if (dim == 3) {
      static const bool whole = std::getenv("QTT_MORTON_PACK_WHOLE") != nullptr;   // A/B: two whole tiles per CTA
      if (pack && two && !whole) {
        const int64_t blocks = nrhs * (N >> kTileBits);
        if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
        morton_pack3_half_kernel<<<int(blocks), kThreads, 0, st>>>(in, out, levels, N);
        return cudaGetLastError();
      }
      if (pack) return two ? launch_tile<3, true, 2>(in, out, levels, N, nrhs, st)
                           : launch_tile<3, true, 1>(in, out, levels, N, nrhs, st);
      return launch_tile<3, false, 1>(in, out, levels, N, nrhs, st);
    }
    if (pack) return two ? launch_tile<2, true, 2>(in, out, levels, N, nrhs, st)
                         : launch_tile<2, true, 1>(in, out, levels, N, nrhs, st);
    return launch_tile<2, false, 1>(in, out, levels, N, nrhs, st);
  } else {
    const int64_t total = N * nrhs;
    int64_t blocks = (total + kThreads - 1) / kThreads;
    blocks = blocks > int64_t(num_sms) * 16 ? int64_t(num_sms) * 16 : blocks;
    if (pack) morton_simple_kernel<true><<<int(blocks), kThreads, 0, st>>>(in, out, dim, levels, total, N);
    else morton_simple_kernel<false><<<int(blocks), kThreads, 0, st>>>(in, out, dim, levels, total, N);
  }
  return cudaGetLastError();
}

}  // namespace qtt
