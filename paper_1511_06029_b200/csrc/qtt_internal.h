// Internal interface between the host planner (qtt_api.cpp) and the kernel
// translation units.  Not part of the public ABI (see include/qtt.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace qtt {

// Kernel variants (also reported through qtt_get_stage).
enum Variant : int { kGeneric = 0, kDmma = 1, kFused = 2 };

// Largest ranks the DMMA level kernel is instantiated for: K = 2 r_in <= 16*kMaxKB,
// 2 * roundup(r_out, 2) <= 8*kMaxNB.
constexpr int kMaxKB = 6;
constexpr int kMaxNB = 12;
constexpr int kDmmaRowGroups = 4;                // 4 x 16 rows = one 64-row sub-tile
constexpr int kDmmaRowsPerSubtile = 16 * kDmmaRowGroups;
// Column groups of consumer warps for a level with NB n8-blocks: 2-3 warps per
// SM sub-partition for the wide levels, fewer for narrow (memory-bound) ones.
__host__ __device__ constexpr int dmma_col_groups(int NB) { return NB >= 9 ? 3 : (NB >= 2 ? 2 : 1); }
__host__ __device__ constexpr int dmma_threads(int NB) { return (kDmmaRowGroups * dmma_col_groups(NB) + 1) * 32; }
constexpr int kMaxStages = 8;

// One level (= one core, PAPER Alg. 2 lines 5-8) as a GEMM over the rotating
// layout:  out[(m + half*(s+i)) * r_out + b] = sum_{j,a} G[a,i,j,b] * in[(2m+j) * r_in + a]
// for rows m < M = nrhs * N/2, s = m / half.
struct LevelArgs {
  const double* in = nullptr;
  double* out = nullptr;
  const double* bpack = nullptr;   // DMMA: packed B fragments (KB*NB*32 double4)
  const double* core = nullptr;    // generic: raw core [a][i][j][b]
  int64_t M = 0;                   // GEMM rows: nrhs * N / 2
  int64_t half = 0;                // N / 2
  int log2_half = 0;               // half = 2^log2_half
  int* tile_counter = nullptr;     // zeroed before the launch; dynamic tile scheduler
  int r_in = 0, r_out = 0;
  int RP = 0;                      // r_out rounded up to even (column padding per half)
  int K = 0;                       // 2 * r_in
  int KB = 0, NB = 0;              // k16 / n8 fragment blocks
  int rep = 1;                     // 64-row sub-tiles per TMA stage
  int stages = 2;                  // TMA pipeline depth
  int grid = 0;
  size_t smem = 0;
};

size_t dmma_smem_bytes(int KB, int NB, int K, int rep, int stages);
cudaError_t dmma_prepare(int KB, int NB, size_t smem);   // sets the max dynamic smem attribute
cudaError_t dmma_occupancy(int KB, int NB, size_t smem, int* ctas_per_sm);
cudaError_t launch_level_dmma(const LevelArgs& a, cudaStream_t st);
cudaError_t launch_level_generic(const LevelArgs& a, cudaStream_t st, int num_sms);

}  // namespace qtt
