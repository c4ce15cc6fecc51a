// Internal runtime of libqtt_b200.so shared by the ABI translation units
// (qtt_api.cpp, qtt_api_ext.cpp, qtt_host_copy.cpp, qtt_runtime.cpp).  Not
// part of the public ABI (include/qtt.h).
#pragma once
#include "../../include/qtt.h"
#include "qtt_internal.h"

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace qtt {
namespace rt {

using qtt::LevelArgs;

// One launch of an apply: levels k0..k1 (a single level, or a merged stage).
struct Stage {
  qtt::StagePlan plan;
  int ctas_per_sm = 1;
  double* d_bpack = nullptr;   // DMMA fragment-packed (super-)core
  double* d_core = nullptr;    // raw core (generic kernel, single level only)
  int64_t* d_coloff = nullptr; // wide stages: output-column offsets of the epilogue (LevelArgs::col_off)
};

struct StageEvents {
  cudaEvent_t start, stop;
  int stage;
};

}  // namespace rt
}  // namespace qtt

using qtt::rt::Stage;
using qtt::rt::StageEvents;

struct qtt_plan {
  int device = 0;
  int num_sms = 0;
  size_t smem_optin = 0;
  int d = 0;
  int64_t N = 0;
  std::vector<int64_t> ranks;
  std::vector<Stage> stages;
  std::vector<double*> d_raw;      // raw cores G_k [a][i][j][b] (compressed matvec)
  // top-bit shard (qtt_create_shard): the handle's d, N, ranks, stages are the
  // local levels 1..d-s; `proj` maps their output onto the 2^s output blocks
  int shard_bits = 0;
  int shard_part = 0;
  Stage proj;
  std::vector<double> proj_W;      // c_{h,part}[alpha] (P x r), kept for the fused exchange
  Stage proj_fused;                // the projection as a wide stage writing into peers
  double** d_peers = nullptr;      // device table of the P receive buffers (qtt_shard_set_peers)
  int64_t max_interior_rank = 0;
  // fused apply (variant kFused, ONE launch per apply): the
  // stage split of the persistent kernel, packed as small stages; used for
  // applies with nrhs <= fused_max_nrhs (0 = never) unless stage timing is on
  std::vector<Stage> fstages;
  int64_t fused_max_nrhs = 0;
  bool ws_header_zero = false;     // the cached workspace's grid-barrier words are 0
  bool fused_on = true;            // qtt_set_fused
  // cached workspace (qtt_apply, qtt_apply_host, shard applies) and the event
  // recorded after the last apply that used it (cross-stream ordering; no
  // caller stream is kept beyond a call)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaEvent_t ws_used = nullptr;
  bool ws_pending = false;
  // cached QTT-order staging vectors (qtt_apply_grid): one allocation, gy = gx + g_elems
  double* gx = nullptr;
  double* gy = nullptr;
  size_t g_elems = 0;
  cudaEvent_t g_used = nullptr;
  bool g_pending = false;
  // cached scratch of the compressed matvec (b's cores, product cores, densify workspace)
  void* cmv = nullptr;
  size_t cmv_bytes = 0;
  // cached staging buffers (qtt_apply_host)
  double* hx = nullptr;
  double* hy = nullptr;
  size_t h_elems = 0;
  cudaEvent_t last = nullptr;
  // CUDA graphs of whole applies, keyed on (x, y, ws, nrhs): one cudaGraphLaunch
  // replaces the memset + per-stage launches (latency-bound small problems)
  struct Graph {
    const double* x;
    double* y;
    void* ws;
    int64_t nrhs;
    cudaGraphExec_t exec;
    int kind;          // 0 per-stage plan, 1 fused launch, 2 fused launch + barrier reset
  };
  std::vector<Graph> graphs;
  cudaStream_t capture_stream = nullptr;
  // qtt_apply_host pipelining: copy stream and chunk events
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> pipe_events;
  unsigned* d_sync = nullptr;      // [kSyncChunks] ready flags + [kSyncChunks] done counters
  unsigned epoch = 0;
  bool timing = false;
  std::vector<StageEvents> pending;
  std::vector<double> stage_ms;
  int timed_applies = 0;
};

// Product of QTT operators applied right to left (qtt_product_create).
struct qtt_product {
  std::vector<qtt_plan*> factors;   // y = F_0 F_1 ... F_{n-1} x; not owned
  int device = 0;
  int64_t N = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaEvent_t ws_used = nullptr;
  bool ws_pending = false;
};

namespace qtt {
namespace rt {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// Workspace layout: [256 B: per-stage tile counters of the dynamic scheduler]
// [buffer 0][buffer 1], each buffer max stage-boundary rank * N * nrhs doubles
// (the ping-pong intermediate y_k of Alg. 2 at the stage boundaries).
constexpr size_t kWsHeader = 256;

struct WideHooks {
  double* const* peers = nullptr;
  int64_t peer_offset = 0;
  const unsigned* ready = nullptr;
  unsigned ready_val = 0;
  int64_t ready_rows = 0;
  unsigned* done = nullptr;
  int64_t done_rows = 0;
};

// B operand of a stage in MMA-fragment order (see qtt_dmma_kernel.cuh):
//   pack[kb][nb][lane][v] = Bmat(kb*16 + 4*(lane%4) + v, nb*8 + lane/4)
// Bmat(kk, n) returns the GEMM operand (0 for padding).
template <class F>
std::vector<double> pack_dmma_fn(const qtt::StagePlan& sp, F bmat) {
  const int KB = sp.KB, NB = sp.NB;
  std::vector<double> out(size_t(KB) * NB * 32 * 4, 0.0);
  for (int kb = 0; kb < KB; ++kb)
    for (int nb = 0; nb < NB; ++nb)
      for (int lane = 0; lane < 32; ++lane)
        for (int v = 0; v < 4; ++v)
          out[((size_t(kb) * NB + nb) * 32 + lane) * 4 + v] = bmat(kb * 16 + 4 * (lane % 4) + v, nb * 8 + lane / 4);
  return out;
}

// B operand of a wide stage, streamed by k-chunk (qtt_wide_kernel.cu):
//   pack[cb][ch][kb][nb][lane][v] = Bmat(ch*BK + kb*16 + 4*(lane%4) + v, (cb*NB + nb)*8 + lane/4)
template <class F>
std::vector<double> pack_wide_fn(const qtt::StagePlan& sp, F bmat) {
  const int NB = sp.NB;
  const size_t chunk = size_t(qtt::kWideKBC) * NB * 32 * 4;
  std::vector<double> out(size_t(sp.ncb) * sp.nchunks * chunk, 0.0);
  for (int cb = 0; cb < sp.ncb; ++cb)
    for (int ch = 0; ch < sp.nchunks; ++ch)
      for (int kb = 0; kb < qtt::kWideKBC; ++kb)
        for (int nb = 0; nb < NB; ++nb)
          for (int lane = 0; lane < 32; ++lane)
            for (int v = 0; v < 4; ++v)
              out[(size_t(cb) * sp.nchunks + ch) * chunk + ((size_t(kb) * NB + nb) * 32 + lane) * 4 + v] =
                  bmat(ch * qtt::kWideBK + kb * 16 + 4 * (lane % 4) + v, (cb * NB + nb) * 8 + lane / 4);
  return out;
}

// B operand of a small stage (qtt_wide_kernel.cu small_dmma_kernel):
//   pack[cb][q][lane][s][nb] = Bmat(q*8 + 2*(lane%4) + s, cb*32 + nb*8 + lane/4)
template <class F>
std::vector<double> pack_small_fn(const qtt::StagePlan& sp, F bmat) {
  std::vector<double> out(size_t(sp.ncb) * sp.nchunks * 32 * 8, 0.0);
  for (int cb = 0; cb < sp.ncb; ++cb)
    for (int q = 0; q < sp.nchunks; ++q)
      for (int lane = 0; lane < 32; ++lane)
        for (int s = 0; s < 2; ++s)
          for (int nb = 0; nb < 4; ++nb)
            out[(((size_t(cb) * sp.nchunks + q) * 32 + lane) * 2 + s) * 4 + nb] =
                bmat(q * qtt::kSmallK + 2 * (lane % 4) + s, cb * qtt::kSmallCols + nb * 8 + lane / 4);
  return out;
}

// B operand of a fused stage (qtt_wide_kernel.cu fused_small_kernel), per
// 32-column block a contiguous run the kernel copies to smem whole:
//   pack[cb][q][s][h][lane][e] = Bmat(q*8 + 2*(lane%4) + s, cb*32 + (2h + e)*8 + lane/4)
template <class F>
std::vector<double> pack_fused_fn(const qtt::StagePlan& sp, F bmat) {
  std::vector<double> out(size_t(sp.ncb) * sp.nchunks * 256, 0.0);
  for (int cb = 0; cb < sp.ncb; ++cb)
    for (int q = 0; q < sp.nchunks; ++q)
      for (int s = 0; s < 2; ++s)
        for (int h = 0; h < 2; ++h)
          for (int lane = 0; lane < 32; ++lane)
            for (int e = 0; e < 2; ++e)
              out[((((size_t(cb) * sp.nchunks + q) * 2 + s) * 2 + h) * 32 + lane) * 2 + e] =
                  bmat(q * qtt::kSmallK + 2 * (lane % 4) + s, cb * qtt::kSmallCols + (2 * h + e) * 8 + lane / 4);
  return out;
}

qtt_status_t from_cuda(cudaError_t e);
bool is_device_ptr(const void* p, int dev = -1);
std::vector<double> super_core(const double* const* cores, const int64_t* ranks, int k0, int k1);
std::vector<double> pack_dmma(const double* W, const qtt::StagePlan& sp);
std::vector<double> pack_wide(const double* W, const qtt::StagePlan& sp);
std::vector<double> pack_small(const double* W, const qtt::StagePlan& sp);
std::vector<double> pack_fused(const double* W, const qtt::StagePlan& sp);
std::vector<double> shard_projection(int d, const int64_t* ranks, const double* const* cores, int s, int g);
size_t ws_buf_bytes(const qtt_plan* h, int64_t nrhs);
size_t ws_bytes_for(const qtt_plan* h, int64_t nrhs);
// Right-hand sides per launch group: every launch keeps N * group <= 2^31 so
// each GEMM row index is a valid 32-bit TMA coordinate; an apply with more
// RHS runs as consecutive groups (the RHS are independent problems, and the
// plan -- split-K included -- does not depend on the group size, so results
// are bitwise those of one launch per RHS).
constexpr int64_t kMaxRowsPerLaunch = int64_t(1) << 31;
inline int64_t rhs_group(const qtt_plan* h, int64_t nrhs) {
  const int64_t g = kMaxRowsPerLaunch / h->N;
  return nrhs < g ? nrhs : (g < 1 ? 1 : g);
}
void free_plan(qtt_plan* h);
qtt_status_t upload_stage(qtt_plan* h, Stage& S, const double* const* cores);
// split-K scratch inside the workspace (enqueue); nullptr = no split
struct SplitScratch {
  double* partial = nullptr;
};
int stage_ksplit(const qtt_plan* h, const Stage& S, int64_t M);
cudaError_t setup_split(const qtt_plan* h, void* ws, int64_t nrhs, cudaStream_t st, SplitScratch* out);
cudaError_t launch_stage(qtt_plan* h, const Stage& S, bool proj, const double* in, double* out, int64_t M,
                         int64_t m_base, int* counter, cudaStream_t st, const WideHooks* hooks = nullptr,
                         const SplitScratch* split = nullptr);
qtt_status_t enqueue(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st,
                     bool fused = false);
qtt_status_t enqueue_graphed(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st,
                             int kind = 0);
// the fused apply (one persistent launch); zero_bar: clear the workspace's
// grid-barrier words first (a workspace not known to hold them at 0)
bool use_fused(const qtt_plan* h, int64_t nrhs);
qtt_status_t enqueue_fused(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st,
                           bool zero_bar, int morton_dim = 0);
// qtt_apply_grid through the fused apply: the Morton gather / scatter happen
// in its first / last stage (qtt_api.cpp); NOT_SUPPORTED when the apply is not fused
qtt_status_t grid_apply_fused(qtt_plan* h, const double* grid_in, double* grid_out, int64_t nrhs, int dim,
                              cudaStream_t st);
// true while `st` is being captured into a CUDA graph (ours or the caller's)
bool stream_is_capturing(cudaStream_t st);
// Grow-only device buffers cached per handle (workspace, grid staging,
// product workspace).  cached_acquire orders `st` after the previous apply
// that used the buffer (its `used` event; skipped while `st` is being
// captured), then -- if `need` exceeds the buffer -- releases the old block on
// `st` itself (so the free follows every earlier user) and allocates the new
// one there; *grew reports that.  A buffer cannot grow during a capture (it
// would belong to the caller's graph): NOT_SUPPORTED.  cached_release records
// `used` on `st` after the apply's last use (skipped while capturing).
qtt_status_t cached_acquire(void** ptr, size_t* bytes, cudaEvent_t* used, bool pending, size_t need,
                            cudaStream_t st, bool capturing, bool* grew);
qtt_status_t cached_release(cudaEvent_t used, bool* pending, cudaStream_t st, bool capturing);
qtt_status_t check_apply_args(qtt_plan* h, const double* x, const double* y, int64_t nrhs);
// qtt_host_copy.cpp
qtt_status_t apply_host_pipelined(qtt_plan* h, const double* x_host, double* y_host, cudaStream_t st);

}  // namespace rt
}  // namespace qtt
