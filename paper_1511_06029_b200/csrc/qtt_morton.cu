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
// Grids smaller than one tile use a per-element kernel.
#include "qtt_internal.h"

#include <cstdint>
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

template <int DIM, bool PACK>
__global__ void __launch_bounds__(kThreads) morton_tile_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                               int levels, int64_t N) {
  constexpr int B = kTileBits / DIM;          // bits per axis inside the tile
  constexpr int R = 1 << B;                   // row length (x extent)
  __shared__ __align__(16) double tile[kTile];

  const int64_t tiles_per_rhs = N >> kTileBits;
  const int64_t s = blockIdx.x / tiles_per_rhs;
  const int64_t tq = blockIdx.x - s * tiles_per_rhs;      // tile index in QTT order
  // tile origin in grid coordinates: the QTT bits above kTileBits, de-interleaved
  int64_t c0[3] = {0, 0, 0};
  for (int l = B; l < levels; ++l)
    for (int a = 0; a < DIM; ++a) c0[a] |= ((tq >> (DIM * (l - B) + a)) & 1) << l;
  const int64_t n = int64_t(1) << levels;
  const int64_t gbase = s * N + (DIM == 3 ? (c0[2] * n + c0[1]) * n + c0[0] : c0[1] * n + c0[0]);
  const int64_t qbase = s * N + (tq << kTileBits);

  // smem slot of local QTT index u
  auto slot_of_u = [](int u) {
    int x = 0, y = 0, z = 0;
#pragma unroll
    for (int l = 0; l < B; ++l) {
      x |= ((u >> (DIM * l)) & 1) << l;
      y |= ((u >> (DIM * l + 1)) & 1) << l;
      if (DIM == 3) z |= ((u >> (DIM * l + 2)) & 1) << l;
    }
    const int row = DIM == 3 ? z * R + y : y;
    return row * R + (x ^ swz<DIM>(row));
  };
  // global offset (from gbase) and smem slot of the e-th element in natural order
  auto grid_of_e = [n](int e, int64_t& goff, int& slot) {
    const int x = e & (R - 1), row = e >> B;      // row = z*R + y (dim 3) or y (dim 2)
    const int y = row & (R - 1), z = row >> B;
    goff = (DIM == 3 ? (int64_t(z) * n + y) * n : int64_t(y) * n) + x;
    slot = row * R + (x ^ swz<DIM>(row));
  };

  // 16-byte accesses on both sides: x pairs (x even, x + 1) stay adjacent under
  // the swizzle (it flips only bits 2-3 of x), and u pairs are x pairs.
  double2* tile2 = reinterpret_cast<double2*>(tile);
  if (PACK) {
#pragma unroll
    for (int e = 2 * threadIdx.x; e < kTile; e += 2 * kThreads) {
      int64_t goff;
      int slot;
      grid_of_e(e, goff, slot);
      tile2[slot >> 1] = __ldcs(reinterpret_cast<const double2*>(in + gbase + goff));
    }
    __syncthreads();
#pragma unroll
    for (int u = 2 * threadIdx.x; u < kTile; u += 2 * kThreads)
      __stcs(reinterpret_cast<double2*>(out + qbase + u), tile2[slot_of_u(u) >> 1]);
  } else {
#pragma unroll
    for (int u = 2 * threadIdx.x; u < kTile; u += 2 * kThreads)
      tile2[slot_of_u(u) >> 1] = __ldcs(reinterpret_cast<const double2*>(in + qbase + u));
    __syncthreads();
#pragma unroll
    for (int e = 2 * threadIdx.x; e < kTile; e += 2 * kThreads) {
      int64_t goff;
      int slot;
      grid_of_e(e, goff, slot);
      __stcs(reinterpret_cast<double2*>(out + gbase + goff), tile2[slot >> 1]);
    }
  }
}

}  // namespace

cudaError_t launch_morton(const double* in, double* out, int dim, int levels, int64_t nrhs, bool pack,
                          cudaStream_t st, int num_sms) {
  const int d = dim * levels;
  const int64_t N = int64_t(1) << d;
  const bool aligned = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const bool tiled = aligned && ((dim == 3 && levels >= 4) || (dim == 2 && levels >= 6));
  if (tiled) {
    const int64_t blocks = nrhs * (N >> kTileBits);
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    if (dim == 3) {
      if (pack) morton_tile_kernel<3, true><<<int(blocks), kThreads, 0, st>>>(in, out, levels, N);
      else morton_tile_kernel<3, false><<<int(blocks), kThreads, 0, st>>>(in, out, levels, N);
    } else {
      if (pack) morton_tile_kernel<2, true><<<int(blocks), kThreads, 0, st>>>(in, out, levels, N);
      else morton_tile_kernel<2, false><<<int(blocks), kThreads, 0, st>>>(in, out, levels, N);
    }
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
