// Internal interface between the host planner (qtt_api.cpp, qtt_plan.cpp) and
// the kernel translation units.  Not part of the public ABI (see include/qtt.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>
#ifdef __CUDACC__
#define QTT_HD __host__ __device__
#else
#define QTT_HD
#endif

namespace qtt {

// Kernel variants (also reported through qtt_get_stage).
//   kGeneric : one thread per output element, any rank, one level per launch.
//   kDmma    : one level per launch on the FP64 tensor cores (DMMA).
//   kMerged  : L >= 2 consecutive levels whose cores were contracted into one
//              super-core at create time, applied as ONE DMMA GEMM per launch;
//              the level intermediates never exist.
//   kWide    : a merged stage whose super-core is too large for shared memory:
//              streamed from L2 in k-chunks next to the A tiles (qtt_wide_kernel.cu).
//   kSmall   : latency-bound small stages: one warp per 16 x 32 output block,
//              operands loaded straight from L2 (no smem staging, no barriers).
//   kDiag    : L consecutive levels whose cores are all diagonal in (i_k, j_k)
//              (block-diagonal in those digits, e.g. the paper's surface-wise
//              block-diagonal BIE factor M): the stage is a batched GEMV,
//              out[(m, ii)][b] = sum_a in[(m, ii)][a] D[ii][a][b], 2 r_in r_out
//              flops per element whatever L (qtt_level_dmma.cu diag_kernel).
//   kFused   : every stage of a latency-bound apply in ONE persistent launch
//              (small-variant warp tiles, grid barriers between stages,
//              intermediates in L2; qtt_wide_kernel.cu fused_small_kernel).
enum Variant : int { kGeneric = 0, kDmma = 1, kMerged = 2, kWide = 3, kSmall = 4, kDiag = 5, kFused = 6 };
constexpr int kDiagMaxROut = 8;                       // r_out of the row-per-lane diagonal kernel
constexpr int kDiagMaxRank = 64;                      // r_in, r_out of any diagonal stage
constexpr int kDiagMaxLevels = 24;
constexpr size_t kDiagMaxCoreDoubles = size_t(1) << 23;   // D = r_in x 2^L x r_out
// small variant: 16-row x 32-column warp tiles, k in steps of 8 (two k4 MMAs
// per 16-byte A load), 4 warps per CTA
constexpr int kSmallRows = 16;
constexpr int kSmallCols = 32;
constexpr int kSmallK = 8;
constexpr int kSmallWarps = 4;

// DMMA kernel instances: K = n_i * r_in <= 16*KB, n_i * roundup(r_out, 2) <= 8*NB.
constexpr int kMaxKB = 8;
constexpr int kMaxNB = 16;
QTT_HD constexpr bool dmma_instantiated(int KB, int NB) {
  return KB >= 1 && NB >= 1 &&
         ((KB <= 6 && NB <= 12) || (KB <= 8 && NB <= 8) || (KB <= 4 && NB <= 16));
}
constexpr int kDmmaRowGroups = 4;                // 4 x 16 rows = one 64-row sub-tile
constexpr int kDmmaRowsPerSubtile = 16 * kDmmaRowGroups;
// Column groups of consumer warps for a stage with NB n8-blocks: 2-3 warps per
// SM sub-partition for the wide stages, fewer for narrow (memory-bound) ones.
#ifndef QTT_CG3_MIN_NB
#define QTT_CG3_MIN_NB 9
#endif
QTT_HD constexpr int dmma_col_groups(int NB) { return NB >= QTT_CG3_MIN_NB ? 3 : (NB >= 2 ? 2 : 1); }
QTT_HD constexpr int dmma_threads(int NB) { return (kDmmaRowGroups * dmma_col_groups(NB) + 1) * 32; }
constexpr int kMaxStages = 8;
constexpr int kBarBytes = 256;   // full[8] + empty[8] mbarriers + tile_id[8]
constexpr int kMaxStageLevels = 10;  // most levels one merged stage may cover

// Wide (streamed super-core) kernel: 64-row tiles, BN = 8*NB columns per
// column block, k-chunks of kWideBK; instances for NB in {4, 8, 12, 16}.
constexpr int kWideKBC = 2;                  // k16 blocks per chunk
constexpr int kWideBK = 16 * kWideKBC;       // 32
// experiment knobs (A/B builds): ring depth, widest column block,
// persistent CTAs per SM of the wide kernel
#ifndef QTT_WIDE_STAGES
#define QTT_WIDE_STAGES 4
#endif
#ifndef QTT_WIDE_NB_CAP
#define QTT_WIDE_NB_CAP 16
#endif
#ifndef QTT_WIDE_CTAS
#define QTT_WIDE_CTAS 1
#endif
constexpr int kWideStages = QTT_WIDE_STAGES;
constexpr size_t kWideMaxCoreBytes = size_t(64) << 20;
QTT_HD constexpr bool wide_instantiated(int NB) { return NB == 4 || NB == 8 || NB == 12 || NB == 16; }

// One stage (L consecutive levels k0..k0+L-1, n_i = 2^L) as a GEMM over the
// rotating layout (PAPER Alg. 2 lines 5-8 applied L times):
//   row m < M = nrhs * N / n_i of the A operand = the n_i * r_in contiguous
//   doubles at in + m * n_i * r_in  (input rows n_i*m .. n_i*m + n_i - 1);
//   out[(m + Q*(s*(n_i-1) + ii)) * r_out + b] = sum_{jj,a} W[a,ii,jj,b] * A[m][jj*r_in + a]
// with Q = N / n_i, s = m / Q (the RHS), W the stage's super-core.  L = 1 is
// one level of Alg. 2 (W = G_k): out row m + (N/2)(s + i_k).
#ifdef QTT_BOUNDS_CHECK
#define QTT_CHECK_OUT(p, ptr, n)                                                                        \
  do {                                                                                                \
    if ((p).out_limit && ((ptr) < (p).out || (ptr) - (p).out + (n) > (p).out_limit)) __trap();       \
  } while (0)
#else
#define QTT_CHECK_OUT(p, ptr, n) \
  do {                           \
  } while (0)
#endif

struct LevelArgs {
  const double* in = nullptr;
  double* out = nullptr;
  const double* bpack = nullptr;   // DMMA: packed B fragments (KB*NB*32 double4)
  const double* core = nullptr;    // generic: raw core [a][i][j][b]
  int64_t M = 0;                   // GEMM rows of this launch: nrhs * N / n_i, or a chunk of them
                                   // (chunks: one RHS only; `in` and `out` are pre-offset)
  int64_t q = 0;                   // Q = N / n_i
  int log2_q = 0;                  // Q = 2^log2_q
  int n_i = 2;                     // 2^L output (and input) digit combinations
  int* tile_counter = nullptr;     // zeroed before the launch; dynamic tile scheduler
  int r_in = 0, r_out = 0;
  int RP = 0;                      // r_out rounded up to even (column padding per ii block)
  int K = 0;                       // n_i * r_in
  int KB = 0, NB = 0;              // k16 / n8 fragment blocks
  int rep = 1;                     // 64-row sub-tiles per TMA stage
  int stages = 2;                  // TMA pipeline depth
  int grid = 0;
  size_t smem = 0;
  // wide variant only
  int nchunks = 1;                 // K / kWideBK
  int ncb = 1;                     // column blocks of 8*NB columns
  int nout = 0;                    // n_i * r_out real output columns (RP = r_out)
  // wide variant, host-copy pipelining (qtt_apply_host): the producer waits for
  // ready[m0 / ready_rows] >= ready_val (written by the copy stream after each
  // H2D chunk) before loading a tile's A rows; each consumer warp adds 1 to
  // done[m0 / done_rows] once its part of a tile is stored
  const unsigned* ready = nullptr;
  unsigned ready_val = 0;
  int64_t ready_rows = 0;
  unsigned* done = nullptr;
  int64_t done_rows = 0;
  // wide variant, fused shard exchange: output column ii (r_out = 1) of row m is
  // stored at peers[ii][m] -- part ii's receive slot for this part (NVLink
  // peer memory on a multi-GPU node)
  double* const* peers = nullptr;
  int64_t peer_offset = 0;         // added to every peers[ii] (this part's slot: part * M)
  // wide variant, split-K (ksplit > 1): tile t = output tile t / ksplit, k-chunks
  // [(t % ksplit) * kcps, ...); partial sums in `partial`, reduced by the next launch
  // debug builds (-DQTT_BOUNDS_CHECK): doubles addressable from `out` (0 = unchecked);
  // every epilogue store traps outside [out, out + out_limit)
  int64_t out_limit = 0;
  // wide variant, plain epilogue: col_off[n] = (ii << log2_q) r_out + b for
  // output column n = ii r_out + b (host-computed, L1-cached), and the tile ->
  // (row tile, column block) split as a multiply-shift (ncb_mul = 0: divide)
  const int64_t* col_off = nullptr;
  uint32_t ncb_mul = 0;
  int ncb_shr = 0;
  int ksplit = 1;
  int kcps = 0;                    // k-chunks per split
  double* partial = nullptr;       // [output tiles][ksplit][consumer warps][split_slot_doubles(NB)]
};

// Host-side stage plan (qtt_plan.cpp): pure function of the rank profile and
// device limits, no CUDA calls.
struct StagePlan {
  int k0 = 1, k1 = 1;              // 1-based levels covered
  int variant = kGeneric;
  int r_in = 0, r_out = 0, n_i = 2;
  int K = 0, KB = 0, NB = 0, RP = 0, rep = 1, stages = 2;
  int nchunks = 1, ncb = 1;        // wide variant
  int ksplit = 1;                  // wide variant: k-split at nrhs = 1 (re-derived per launch)
  size_t smem = 0;
  double est_seconds = 0;          // cost-model estimate at nrhs = 1
};

size_t dmma_smem_bytes(int KB, int NB, int K, int rep, int stages);
// Tiling of a DMMA stage; false if it does not fit smem_optin.
bool dmma_tiling(int K, int KB, int NB, size_t smem_optin, int* rep, int* stages, size_t* smem);
// diag[k-1] != 0: core k is diagonal in (i_k, j_k) (nullptr: none known)
// rows = nrhs * N the estimates are made at (0: N, one RHS)
std::vector<StagePlan> plan_stages(int d, const int64_t* ranks, size_t smem_optin, int max_stage_levels,
                                   const unsigned char* diag = nullptr, int64_t rows = 0);
double plan_seconds(const std::vector<StagePlan>& p);   // sum of the stage estimates
// one fused stage's shape and estimate at `rows` input rows (-1: too large)
double fused_stage_seconds(const int64_t* ranks, int k0, int k1, double rows, StagePlan* sp);
double fused_launch_seconds();
// fused apply (variant kFused): the stage split of one persistent launch at
// `rows` = nrhs * N GEMM input rows, and its estimated time (*est; +inf and an
// empty plan when none fits)
std::vector<StagePlan> plan_stages_fused(int d, const int64_t* ranks, int max_stage_levels, int64_t rows,
                                         double* est);
bool projection_plan(int r, int s, size_t smem_optin, StagePlan* sp);
bool projection_plan_wide(int r, int s, size_t smem_optin, StagePlan* sp);   // fused exchange

cudaError_t dmma_prepare(int KB, int NB, size_t smem);   // sets the max dynamic smem attribute
cudaError_t dmma_occupancy(int KB, int NB, size_t smem, int* ctas_per_sm);
cudaError_t launch_level_dmma(const LevelArgs& a, cudaStream_t st);
cudaError_t launch_level_generic(const LevelArgs& a, cudaStream_t st, int num_sms);
// diagonal stage: a.core = D [n_i][r_in][r_out], a.M = GEMM rows (nrhs N / n_i)
cudaError_t launch_diag(const LevelArgs& a, cudaStream_t st, int num_sms);
size_t wide_smem_bytes(int NB);
#ifndef QTT_WIDE_CG4_MIN_NB
#define QTT_WIDE_CG4_MIN_NB 16
#endif
// column groups of the wide kernel's consumer warps: 4 (16 warps, 4 n-blocks
// each, 96 registers, no spills) for NB = 16 -- measured 1-3.5% faster than
// 3 groups of 6/5/5 n-blocks (c3 stages, c4 top, large ranks; A/B r01ay)
QTT_HD constexpr int wide_col_groups(int NB) {
  return (NB >= QTT_WIDE_CG4_MIN_NB && NB % 4 == 0) ? 4 : dmma_col_groups(NB);
}
QTT_HD constexpr int wide_threads(int NB) { return (kDmmaRowGroups * wide_col_groups(NB) + 1) * 32; }
QTT_HD constexpr int wide_consumer_warps(int NB) { return kDmmaRowGroups * wide_col_groups(NB); }
// split-K partial of one consumer warp: 16 rows x (widest column group) x 8 columns
QTT_HD constexpr int split_slot_doubles(int NB) {
  return ((NB + wide_col_groups(NB) - 1) / wide_col_groups(NB)) * 128;
}
// k-split of a wide stage with `tiles` output tiles of `nchunks` k-chunks on
// `sms` SMs: minimises waves x (chunks per split + epilogue), 1 = no split
// (qtt_plan.cpp)
int wide_ksplit(int64_t tiles, int nchunks, int sms);
// diagnostics: QTT_NO_PDL=1 launches the stage kernels without programmatic
// dependent launch, QTT_NO_SPLIT=1 plans no split-K stages
bool pdl_enabled();
bool split_enabled();
cudaError_t wide_prepare(int NB, size_t smem);
cudaError_t launch_wide(const LevelArgs& a, cudaStream_t st);
// small variant (qtt_wide_kernel.cu): a.ncb = 32-column blocks, a.nchunks = k-steps of 8,
// a.bpack = pack_small layout
cudaError_t launch_small(const LevelArgs& a, cudaStream_t st);
// fused apply (variant kFused): the stages of one apply in one cooperative launch
constexpr int kFusedWarps = 8;        // warps per CTA (two per SM sub-partition)
constexpr int kFusedMaxStages = 6;
constexpr size_t kFusedMaxCoreBytes = size_t(4) << 20;   // a fused stage's packed super-core, read from L2
constexpr size_t kFusedMaxBBytes = size_t(128) << 10;    // one column block of it in smem: K <= 512
constexpr size_t kFusedMaxL2Bytes = size_t(40) << 20;    // both intermediate buffers of a fused apply
constexpr size_t kFusedBarOffset = 192;                  // grid-barrier words in the workspace header
struct FusedStage {
  const double* in = nullptr;
  double* out = nullptr;
  const double* bpack = nullptr;   // pack_small layout
  int64_t M = 0;                   // GEMM rows: nrhs * N / n_i
  int64_t out_limit = 0;           // QTT_BOUNDS_CHECK builds
  int log2_q = 0, n_i = 2, r_out = 0, nout = 0, K = 0, nchunks = 0, ncb = 0;
  int ks = 1;                      // warps per tile (intra-CTA split of the k-steps; 1, 2, 4 or 8)
  // Morton order fused into the grid apply (qtt_apply_grid): the last stage
  // scatters its output into a natural-order grid (mout_dim; 0 = QTT order;
  // levels per axis = log2n / dim).  The gather is FusedArgs' pre-pass.
  int mout_dim = 0, log2n = 0;
  int runs = 0;                    // run-wise smem epilogue (r_out | 32, Q % 16 == 0, QTT-order output)
  // host-computed work decomposition (no integer division in the kernel):
  int mtiles = 0;                  // 16-row tiles (M + 15) / 16
  int rgroups = 0;                 // row groups of kFusedWarps / ks tiles; units = rgroups * ncb
  int units = 0;
  uint32_t rg_mul = 0;             // u / rgroups = rg_mul ? umulhi(u, rg_mul) >> rg_shr : u >> rg_shr
  int rg_shr = 0;
  int cps = 0;                     // k-steps per split-K part, ceil(nchunks / ks)
  int lks = 0;                     // log2 ks
  int in_dim = 0;                  // the A rows come from a natural-order grid (fused grid apply, stage 0):
                                   // each 16-byte A load gathers two adjacent grid points (Morton, R18)
  int lr = 0;                      // log2 r_out (run-wise epilogue)
};
struct FusedArgs {
  FusedStage st[kFusedMaxStages];
  int nstages = 0;
  unsigned* bar = nullptr;         // arrival counter, 0 at launch (left at 0 by every launch)
  size_t smem = 0;                 // dynamic smem: the largest super-core block (K x 32 doubles)
  int repeat = 1;                  // diagnostic (QTT_FUSED_REPEAT): run every stage this many times
  int early_trigger = 1;           // griddepcontrol.launch_dependents at the last stage (QTT_FUSED_NO_TRIGGER=1: off)
  // fused grid apply: a first pass gathers the natural-order grid pre_src into
  // QTT order at pre_dst (each element once, stores coalesced), then a grid
  // barrier; the stages read pre_dst (the last stage scatters: mout_dim)
  const double* pre_src = nullptr;
  double* pre_dst = nullptr;
  int pre_dim = 0, pre_log2n = 0;
  int64_t pre_total = 0;
  unsigned long long* prof = nullptr;   // diagnostic (QTT_FUSED_PROFILE): per CTA, %globaltimer
                                        // at start and after each stage's tiles / barrier, then for
                                        // the CTA's first unit of each stage: start, super-core block
                                        // in smem, MMAs done, tile stored
};
constexpr int kFusedProfBase = 2 * kFusedMaxStages + 2 + 4 * kFusedMaxStages;
// then per stage and warp of the CTA's first unit: A fragment arrived, MMAs done,
// past the split-K __syncthreads, tile stored (ns, %globaltimer)
constexpr int kFusedProfSlots = kFusedProfBase + kFusedMaxStages * kFusedWarps * 4;
cudaError_t fused_prepare();   // sets the kernel's max dynamic smem
bool fused_cooperative();       // QTT_FUSED_COOP=1: launch with the cooperative attribute
cudaError_t launch_fused(const FusedArgs& a, int grid, cudaStream_t st, bool pdl = true);
// natural-grid offset of QTT index q < 2^30 within one RHS (Morton order,
// DESIGN.md R18: QTT bit dim*l + a = bit l of coordinate a; x fastest): the
// coordinates are every dim-th bit of q, compacted with mask-and-shift steps
// (constant time, registers only)
QTT_HD inline uint32_t morton_compact3(uint32_t v) {
  v &= 0x09249249u;
  v = (v ^ (v >> 2)) & 0x030c30c3u;
  v = (v ^ (v >> 4)) & 0x0300f00fu;
  v = (v ^ (v >> 8)) & 0xff0000ffu;
  v = (v ^ (v >> 16)) & 0x000003ffu;
  return v;
}
QTT_HD inline uint32_t morton_compact2(uint32_t v) {
  v &= 0x55555555u;
  v = (v ^ (v >> 1)) & 0x33333333u;
  v = (v ^ (v >> 2)) & 0x0f0f0f0fu;
  v = (v ^ (v >> 4)) & 0x00ff00ffu;
  v = (v ^ (v >> 8)) & 0x0000ffffu;
  return v;
}
QTT_HD inline int64_t morton_natural(int64_t q, int dim, int levels) {
  const uint32_t u = uint32_t(q);
  if (dim == 3)
    return int64_t(morton_compact3(u)) | (int64_t(morton_compact3(u >> 1)) << levels) |
           (int64_t(morton_compact3(u >> 2)) << (2 * levels));
  if (dim == 2) return int64_t(morton_compact2(u)) | (int64_t(morton_compact2(u >> 1)) << levels);
  return q;
}
// y[s][c] = sum_g recv[g][s][c] (fixed order g = 0..parts-1), qtt_wide_kernel.cu
cudaError_t launch_shard_reduce(const double* recv, double* y, int parts, int64_t count, cudaStream_t st,
                                int num_sms);
// QTT-compressed matvec cores and TT-vector densification, qtt_compressed.cu
cudaError_t compressed_cores(int d, const int64_t* ra, const double* const* dG, const int64_t* rb,
                             const double* const* dV, double* const* dC, cudaStream_t st, int num_sms);
size_t densify_workspace_bytes(int d, const int64_t* R);
cudaError_t tt_densify(int d, const int64_t* R, const double* const* dH, double* out, void* ws, cudaStream_t st,
                       int num_sms, size_t smem_optin);
// Morton pack (natural grid -> QTT order) or unpack, qtt_morton.cu
cudaError_t launch_morton(const double* in, double* out, int dim, int levels, int64_t nrhs, bool pack,
                          cudaStream_t st, int num_sms);

}  // namespace qtt
