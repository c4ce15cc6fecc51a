// C ABI of libqtt_b200.so (declared and documented in include/qtt.h).
//
// Host side of the QTT apply: argument validation, core packing and super-core
// contraction, the stage plan (B4, qtt_plan.cpp), workspace
// management and launches.  The
// arithmetic of PAPER.md Alg. 2 runs entirely in the kernels
// (qtt_level_dmma.cu); nothing here touches vector data.
#include "../../include/qtt.h"
#include "qtt_internal.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

namespace {

using qtt::LevelArgs;

// One launch of an apply: levels k0..k1 (a single level, or a merged stage).
struct Stage {
  qtt::StagePlan plan;
  int ctas_per_sm = 1;
  double* d_bpack = nullptr;   // DMMA fragment-packed (super-)core
  double* d_core = nullptr;    // raw core (generic kernel, single level only)
};

struct StageEvents {
  cudaEvent_t start, stop;
  int stage;
};

}  // namespace

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
  int64_t max_interior_rank = 0;
  // cached workspace (qtt_apply)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaStream_t ws_stream = nullptr;
  // stream of the last apply that used the cached workspace (cross-stream ordering)
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  // cached QTT-order staging vectors (qtt_apply_grid)
  double* gx = nullptr;
  double* gy = nullptr;
  size_t g_elems = 0;
  cudaStream_t g_stream = nullptr;
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
  cudaStream_t ws_stream = nullptr;
};

namespace {

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

qtt_status_t from_cuda(cudaError_t e) {
  if (e == cudaSuccess) return QTT_SUCCESS;
  if (std::getenv("QTT_DEBUG")) std::fprintf(stderr, "qtt: CUDA error %s\n", cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return QTT_ERROR_OUT_OF_MEMORY;
  }
  return QTT_ERROR_CUDA;
}

// Super-core of levels k0..k1 (PAPER Eq. TTdeccores P:519-523 restricted to the
// stage's digits; qtt_plan.cpp): W[a][ii][jj][b], ii/jj = the stage's output /
// input digits, first level least significant.  Contracted from the narrow
// end of the stage (the rank-1 side of a boundary stage): left to right costs
// sum_l r_in 4^l r_l r_{l+1}, right to left sum_l r_l r_{l+1} 4^(L-l) r_out
// multiply-adds; fp64 accumulation (R17), inner loops contiguous.
std::vector<double> super_core(const double* const* cores, const int64_t* ranks, int k0, int k1) {
  const int L = k1 - k0 + 1;
  const int64_t r_in = ranks[k0 - 1], r_out = ranks[k1];
  double lr = 0, rl = 0;
  for (int l = 1; l < L; ++l) {
    lr += double(r_in) * std::ldexp(1.0, 2 * l) * double(ranks[k0 - 1 + l]) * double(ranks[k0 + l]);
    rl += double(ranks[k1 - l - 1]) * double(ranks[k1 - l]) * std::ldexp(1.0, 2 * l) * double(r_out);
  }
  if (lr <= rl) {
    // left to right: V[a][ii + n i][jj + n j][b] = sum_c W[a][ii][jj][c] G[c][i][j][b]
    const int r0 = int(r_in);
    std::vector<double> W(cores[k0 - 1], cores[k0 - 1] + size_t(r0) * 4 * ranks[k0]);
    int n_i = 2;
    int rc = int(ranks[k0]);
    for (int k = k0 + 1; k <= k1; ++k) {
      const double* G = cores[k - 1];
      const int rb = int(ranks[k]);
      const int n2 = 2 * n_i;
      std::vector<double> V(size_t(r0) * n2 * n2 * rb, 0.0);
      for (int a = 0; a < r0; ++a)
        for (int ii = 0; ii < n_i; ++ii)
          for (int jj = 0; jj < n_i; ++jj)
            for (int c = 0; c < rc; ++c) {
              const double w = W[((size_t(a) * n_i + ii) * n_i + jj) * rc + c];
              if (w == 0.0) continue;
              for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) {
                  const double* g = G + ((size_t(c) * 2 + i) * 2 + j) * rb;
                  double* v = &V[((size_t(a) * n2 + ii + n_i * i) * n2 + jj + n_i * j) * rb];
                  for (int b = 0; b < rb; ++b) v[b] = std::fma(w, g[b], v[b]);
                }
            }
      W.swap(V);
      n_i = n2;
      rc = rb;
    }
    return W;
  }
  // right to left: U[c][ii][jj][b] over levels k+1..k1; prepend level k as the
  // least significant digit: V[a][i + 2 ii][j + 2 jj][b] = sum_c G_k[a][i][j][c] U[c][ii][jj][b]
  const int ro = int(r_out);
  std::vector<double> U(cores[k1 - 1], cores[k1 - 1] + size_t(ranks[k1 - 1]) * 4 * ro);
  int n_i = 2;
  for (int k = k1 - 1; k >= k0; --k) {
    const double* G = cores[k - 1];
    const int ra = int(ranks[k - 1]), rc = int(ranks[k]);
    const int n2 = 2 * n_i;
    std::vector<double> V(size_t(ra) * n2 * n2 * ro, 0.0);
    for (int a = 0; a < ra; ++a)
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
          for (int c = 0; c < rc; ++c) {
            const double g = G[((size_t(a) * 2 + i) * 2 + j) * rc + c];
            if (g == 0.0) continue;
            const double* u = &U[size_t(c) * n_i * n_i * ro];
            for (int ii = 0; ii < n_i; ++ii)
              for (int jj = 0; jj < n_i; ++jj) {
                double* v = &V[((size_t(a) * n2 + i + 2 * ii) * n2 + j + 2 * jj) * ro];
                const double* uu = u + (size_t(ii) * n_i + jj) * ro;
                for (int b = 0; b < ro; ++b) v[b] = std::fma(g, uu[b], v[b]);
              }
          }
    U.swap(V);
    n_i = n2;
  }
  return U;
}

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

// Stage super-core W[a][ii][jj][b] as the DMMA B operand:
//   Bmat[kk][n], kk = jj*r_in + a (the column-merged index of Alg. 2 line 6),
//   n = ii*RP + b (the row-separated output, Alg. 2 line 8), value W[a,ii,jj,b].
std::vector<double> pack_dmma(const double* W, const qtt::StagePlan& sp) {
  const int RP = sp.RP, r_in = sp.r_in, r_out = sp.r_out, n_i = sp.n_i, K = sp.K;
  return pack_dmma_fn(sp, [=](int kk, int n) {
    if (kk >= K) return 0.0;
    const int jj = kk / r_in, a = kk % r_in;
    const int ii = n / RP, b = n % RP;
    return (ii < n_i && b < r_out) ? W[((size_t(a) * n_i + ii) * n_i + jj) * r_out + b] : 0.0;
  });
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

// Wide stage: Bmat[jj*r_in + a][ii*r_out + b] = W[a,ii,jj,b] (no column padding per ii).
std::vector<double> pack_wide(const double* W, const qtt::StagePlan& sp) {
  const int r_in = sp.r_in, r_out = sp.r_out, n_i = sp.n_i, K = sp.K, nout = sp.n_i * sp.r_out;
  return pack_wide_fn(sp, [=](int kk, int n) {
    if (kk >= K || n >= nout) return 0.0;
    const int jj = kk / r_in, a = kk % r_in;
    const int ii = n / r_out, b = n % r_out;
    return W[((size_t(a) * n_i + ii) * n_i + jj) * r_out + b];
  });
}

// Top-bit sharding: projection vectors of part g onto every
// output block h, c_{h,g}[alpha] = [G_{d-s+1}(alpha, h_1, g_1, :) ... G_d(:, h_s, g_s, 0)],
// written as Wp[h * r + alpha], r = ranks[d-s].
std::vector<double> shard_projection(int d, const int64_t* ranks, const double* const* cores, int s, int g) {
  const int P = 1 << s;
  const int r = int(ranks[d - s]);
  std::vector<double> Wp(size_t(P) * r, 0.0);
  for (int h = 0; h < P; ++h) {
    // right to left: v over the bond below level k
    std::vector<double> v(1, 1.0);
    for (int l = s; l >= 1; --l) {
      const int k = d - s + l;                       // 1-based level
      const int hb = (h >> (l - 1)) & 1, gb = (g >> (l - 1)) & 1;
      const int ra = int(ranks[k - 1]), rb = int(ranks[k]);
      const double* G = cores[k - 1];
      std::vector<double> u(ra, 0.0);
      for (int a = 0; a < ra; ++a) {
        double acc = 0.0;
        for (int b = 0; b < rb; ++b) acc = std::fma(G[((size_t(a) * 2 + hb) * 2 + gb) * rb + b], v[b], acc);
        u[a] = acc;
      }
      v.swap(u);
    }
    for (int a = 0; a < r; ++a) Wp[size_t(h) * r + a] = v[a];
  }
  return Wp;
}

// Device (or managed) memory; with dev >= 0 also on that device (a kernel of a
// handle on device A must not touch device B's memory).
bool is_device_ptr(const void* p, int dev = -1) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeManaged) return true;
  return at.type == cudaMemoryTypeDevice && (dev < 0 || at.device == dev);
}

// Workspace layout: [256 B: per-stage tile counters of the dynamic scheduler]
// [buffer 0][buffer 1], each buffer max stage-boundary rank * N * nrhs doubles
// (the ping-pong intermediate y_k of Alg. 2 at the stage boundaries).
constexpr size_t kWsHeader = 256;

size_t ws_buf_bytes(const qtt_plan* h, int64_t nrhs) {
  if (h->stages.size() <= 1 && h->shard_bits == 0) return 0;
  const size_t one = size_t(h->max_interior_rank) * size_t(h->N) * size_t(nrhs) * sizeof(double);
  return (one + 255) / 256 * 256;
}

size_t ws_bytes_for(const qtt_plan* h, int64_t nrhs) { return kWsHeader + 2 * ws_buf_bytes(h, nrhs); }

void free_plan(qtt_plan* h) {
  for (auto& S : h->stages) {
    if (S.d_bpack) cudaFree(S.d_bpack);
    if (S.d_core) cudaFree(S.d_core);
  }
  for (double* p : h->d_raw)
    if (p) cudaFree(p);
  if (h->proj.d_bpack) cudaFree(h->proj.d_bpack);
  if (h->ws) cudaFree(h->ws);
  if (h->gx) cudaFree(h->gx);
  if (h->gy) cudaFree(h->gy);
  if (h->hx) cudaFree(h->hx);
  if (h->hy) cudaFree(h->hy);
  for (auto& e : h->pending) {
    cudaEventDestroy(e.start);
    cudaEventDestroy(e.stop);
  }
  if (h->last) cudaEventDestroy(h->last);
  for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
  if (h->capture_stream) cudaStreamDestroy(h->capture_stream);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  for (auto& e : h->pipe_events) cudaEventDestroy(e);
  if (h->d_sync) cudaFree(h->d_sync);
  delete h;
}

qtt_status_t upload_stage(qtt_plan* h, Stage& S, const double* const* cores) {
  const qtt::StagePlan& sp = S.plan;
  if (sp.variant == qtt::kGeneric) {
    const size_t core_elems = size_t(sp.r_in) * 4 * sp.r_out;
    cudaError_t e = cudaMalloc(&S.d_core, core_elems * sizeof(double));
    if (e != cudaSuccess) return from_cuda(e);
    return from_cuda(cudaMemcpy(S.d_core, cores[sp.k0 - 1], core_elems * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (sp.variant == qtt::kWide) {
    cudaError_t e = qtt::wide_prepare(sp.NB, h->smem_optin);
    if (e != cudaSuccess) return from_cuda(e);
    S.ctas_per_sm = 1;
    const std::vector<double> W = super_core(cores, h->ranks.data(), sp.k0, sp.k1);
    const std::vector<double> pk = pack_wide(W.data(), sp);
    e = cudaMalloc(&S.d_bpack, pk.size() * sizeof(double));
    if (e != cudaSuccess) return from_cuda(e);
    return from_cuda(cudaMemcpy(S.d_bpack, pk.data(), pk.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  // The attribute is per kernel instance and shared by every stage (and plan)
  // that uses it, so raise it to the device maximum rather than this stage's need.
  cudaError_t e = qtt::dmma_prepare(sp.KB, sp.NB, h->smem_optin);
  if (e != cudaSuccess) return from_cuda(e);
  int occ = 0;
  e = qtt::dmma_occupancy(sp.KB, sp.NB, sp.smem, &occ);
  if (e != cudaSuccess) return from_cuda(e);
  S.ctas_per_sm = std::max(1, occ);
  std::vector<double> pk;
  if (sp.k0 == sp.k1) {
    pk = pack_dmma(cores[sp.k0 - 1], sp);
  } else {
    const std::vector<double> W = super_core(cores, h->ranks.data(), sp.k0, sp.k1);
    pk = pack_dmma(W.data(), sp);
  }
  e = cudaMalloc(&S.d_bpack, pk.size() * sizeof(double));
  if (e != cudaSuccess) return from_cuda(e);
  return from_cuda(cudaMemcpy(S.d_bpack, pk.data(), pk.size() * sizeof(double), cudaMemcpyHostToDevice));
}

// One launch of stage S over GEMM rows [m_base, m_base + M) (all rows: m_base = 0,
// M = nrhs * N / n_i).  `in` points at the stage input's row 0.  A chunk
// (m_base > 0) must lie in the first RHS: there every output row is
// m + Q ii, so offsetting `out` by m_base rows is exact.
struct WideHooks {
  const unsigned* ready = nullptr;
  unsigned ready_val = 0;
  int64_t ready_rows = 0;
  unsigned* done = nullptr;
  int64_t done_rows = 0;
};

cudaError_t launch_stage(qtt_plan* h, const Stage& S, bool proj, const double* in, double* out, int64_t M,
                         int64_t m_base, int* counter, cudaStream_t st, const WideHooks* hooks = nullptr) {
  const qtt::StagePlan& sp = S.plan;
  const int L = proj ? 0 : sp.k1 - sp.k0 + 1;
  LevelArgs a;
  a.in = in + m_base * sp.K;
  a.out = out + m_base * sp.r_out;
  a.bpack = S.d_bpack;
  a.core = S.d_core;
  a.n_i = sp.n_i;
  a.log2_q = h->d - L;
  a.q = int64_t(1) << a.log2_q;
  a.M = M;
  a.tile_counter = counter;
  a.r_in = sp.r_in;
  a.r_out = sp.r_out;
  a.RP = sp.RP;
  a.K = sp.K;
  a.KB = sp.KB;
  a.NB = sp.NB;
  a.rep = sp.rep;
  a.stages = sp.stages;
  a.smem = sp.smem;
  a.nchunks = sp.nchunks;
  a.ncb = sp.ncb;
  a.nout = sp.n_i * sp.r_out;
  if (hooks) {
    a.ready = hooks->ready;
    a.ready_val = hooks->ready_val;
    a.ready_rows = hooks->ready_rows;
    a.done = hooks->done;
    a.done_rows = hooks->done_rows;
  }
  cudaError_t e;
  if (sp.variant == qtt::kWide) {
    const int64_t tiles = (a.M + qtt::kDmmaRowsPerSubtile - 1) / qtt::kDmmaRowsPerSubtile * sp.ncb;
    a.grid = int(std::min<int64_t>(tiles, int64_t(h->num_sms)));
    e = qtt::launch_wide(a, st);
  } else if (sp.variant != qtt::kGeneric) {
    const int64_t rows_per_stage = int64_t(qtt::kDmmaRowsPerSubtile) * sp.rep;
    const int64_t tiles = (a.M + rows_per_stage - 1) / rows_per_stage;
    a.grid = int(std::min<int64_t>(tiles, int64_t(h->num_sms) * S.ctas_per_sm));
    e = qtt::launch_level_dmma(a, st);
  } else {
    e = qtt::launch_level_generic(a, st, h->num_sms);
  }
  if (e != cudaSuccess && std::getenv("QTT_DEBUG"))
    std::fprintf(stderr, "qtt: stage (levels %d-%d, variant %d, KB %d NB %d smem %zu grid %d) launch failed: %s\n",
                 sp.k0, sp.k1, sp.variant, sp.KB, sp.NB, a.smem, a.grid, cudaGetErrorString(e));
  return e;
}

qtt_status_t enqueue(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st) {
  unsigned char* base = static_cast<unsigned char*>(ws);
  int* counters = reinterpret_cast<int*>(base);
  const size_t bb = ws_buf_bytes(h, nrhs);
  double* buf[2] = {reinterpret_cast<double*>(base + kWsHeader), reinterpret_cast<double*>(base + kWsHeader + bb)};
  cudaError_t me = cudaMemsetAsync(counters, 0, kWsHeader, st);
  if (me != cudaSuccess) return from_cuda(me);
  const double* in = x;
  const int nloc = int(h->stages.size());
  const int ns = nloc + (h->shard_bits ? 1 : 0);
  for (int si = 0; si < ns; ++si) {
    const bool proj = si == nloc;                  // shard projection stage
    const Stage& S = proj ? h->proj : h->stages[si];
    double* out = (si == ns - 1) ? y : buf[si & 1];
    StageEvents ev{};
    if (h->timing && !proj) {
      ev.stage = si;
      if (cudaEventCreate(&ev.start) != cudaSuccess || cudaEventCreate(&ev.stop) != cudaSuccess)
        return QTT_ERROR_CUDA;
      cudaEventRecord(ev.start, st);
    }
    const int L = proj ? 0 : S.plan.k1 - S.plan.k0 + 1;
    const int64_t M = nrhs * (int64_t(1) << (h->d - L));
    const cudaError_t e = launch_stage(h, S, proj, in, out, M, 0, counters + si, st);
    if (e != cudaSuccess) return from_cuda(e);
    if (h->timing && !proj) {
      cudaEventRecord(ev.stop, st);
      h->pending.push_back(ev);
    }
    in = out;
  }
  if (h->timing) h->timed_applies++;
  if (st != h->capture_stream) cudaEventRecord(h->last, st);
  return QTT_SUCCESS;
}

// Driver stream memory operations (no libcuda link): the copy stream signals
// "H2D chunk c landed" by writing a flag the first stage's producer polls, and
// waits on counters the last stage's consumers bump before each D2H chunk.
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamMemOps {
  WriteValueFn write = nullptr;
  WaitValueFn wait = nullptr;
};
const StreamMemOps& stream_mem_ops() {
  static const StreamMemOps ops = [] {
    StreamMemOps o;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.write = reinterpret_cast<WriteValueFn>(f);
    f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.wait = reinterpret_cast<WaitValueFn>(f);
    if (!o.write || !o.wait) o.write = nullptr, o.wait = nullptr;
    cudaGetLastError();
    return o;
  }();
  return ops;
}

constexpr int kSyncChunks = 32;

// qtt_apply_host with ONE launch per stage when the first and last stages are
// wide: the first stage's producer waits per tile for its x chunk's flag
// (written by the copy stream after the chunk's H2D), the last stage's
// consumers count stored tiles per chunk and the copy stream starts each
// chunk's D2H as soon as its count is complete.  Exposed copy time: one
// chunk each way (1/32 of x and of y).
qtt_status_t apply_host_flagged(qtt_plan* h, const double* x_host, double* y_host, cudaStream_t st) {
  const StreamMemOps& ops = stream_mem_ops();
  const int ns = int(h->stages.size());
  const Stage& S0 = h->stages.front();
  const Stage& SL = h->stages.back();
  if (!h->d_sync) {
    cudaError_t e = cudaMalloc(&h->d_sync, 2 * kSyncChunks * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(h->d_sync, 0, 2 * kSyncChunks * sizeof(unsigned));
    if (e != cudaSuccess) return from_cuda(e);
  }
  unsigned* ready = h->d_sync;
  unsigned* done = h->d_sync + kSyncChunks;
  const unsigned epoch = ++h->epoch;
  unsigned char* base = static_cast<unsigned char*>(h->ws);
  int* counters = reinterpret_cast<int*>(base);
  const size_t bb = ws_buf_bytes(h, 1);
  double* buf[2] = {reinterpret_cast<double*>(base + kWsHeader), reinterpret_cast<double*>(base + kWsHeader + bb)};
  cudaStream_t cs = h->copy_stream;
  cudaEvent_t* ev = h->pipe_events.data();
  // rows per chunk: multiples of the 64-row tiles
  auto rows_per_chunk = [](int64_t M) { return std::max<int64_t>(64, (M / kSyncChunks + 63) / 64 * 64); };
  const int L0 = S0.plan.k1 - S0.plan.k0 + 1, LL = SL.plan.k1 - SL.plan.k0 + 1;
  const int64_t M0 = int64_t(1) << (h->d - L0), ML = int64_t(1) << (h->d - LL);
  const int64_t c0 = rows_per_chunk(M0), cl = rows_per_chunk(ML);
  cudaError_t e = cudaMemsetAsync(counters, 0, kWsHeader, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(done, 0, kSyncChunks * sizeof(unsigned), st);
  if (e == cudaSuccess) e = cudaEventRecord(ev[0], st);        // prior work + resets done
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[0], 0);
  if (e != cudaSuccess) return from_cuda(e);
  for (int64_t m0 = 0; m0 < M0; m0 += c0) {                     // x chunks -> ready flags
    const int64_t m1 = std::min(M0, m0 + c0);
    const size_t off = size_t(m0) << L0, cnt = size_t(m1 - m0) << L0;
    e = cudaMemcpyAsync(h->hx + off, x_host + off, cnt * sizeof(double), cudaMemcpyHostToDevice, cs);
    if (e != cudaSuccess) return from_cuda(e);
    if (ops.write(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(ready + m0 / c0), epoch, 0) !=
        CUDA_SUCCESS)
      return QTT_ERROR_CUDA;
  }
  const double* in = h->hx;
  for (int si = 0; si < ns; ++si) {
    const Stage& S = h->stages[si];
    const int L = S.plan.k1 - S.plan.k0 + 1;
    const int64_t M = int64_t(1) << (h->d - L);
    double* out = (si == ns - 1) ? h->hy : buf[si & 1];
    WideHooks hk;
    if (si == 0) {
      hk.ready = ready;
      hk.ready_val = epoch;
      hk.ready_rows = c0;
    }
    if (si == ns - 1) {
      hk.done = done;
      hk.done_rows = cl;
    }
    e = launch_stage(h, S, false, in, out, M, 0, counters + si, st, (si == 0 || si == ns - 1) ? &hk : nullptr);
    if (e != cudaSuccess) return from_cuda(e);
    in = out;
  }
  // y chunks: rows [m0, m1) of every output block ii, once all their tiles are stored
  const int cw = 4 * qtt::dmma_col_groups(SL.plan.NB);        // consumer warps per CTA
  for (int64_t m0 = 0; m0 < ML; m0 += cl) {
    const int64_t m1 = std::min(ML, m0 + cl);
    const unsigned target = unsigned(((m1 - m0 + 63) / 64) * SL.plan.ncb * cw);
    if (ops.wait(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(done + m0 / cl), target,
                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return QTT_ERROR_CUDA;
    e = cudaMemcpy2DAsync(y_host + m0, size_t(ML) * sizeof(double), h->hy + m0, size_t(ML) * sizeof(double),
                          size_t(m1 - m0) * sizeof(double), size_t(1) << LL, cudaMemcpyDeviceToHost, cs);
    if (e != cudaSuccess) return from_cuda(e);
  }
  e = cudaEventRecord(ev[1], cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[1], 0);
  if (e == cudaSuccess) e = cudaEventRecord(h->last, st);
  return from_cuda(e);
}

// qtt_apply_host for one RHS with the host<->device copies overlapped with the
// first and last stages: the first stage runs in row chunks, chunk c waiting
// only for its slice of x (H2D on a copy stream); the last stage runs in row
// chunks, each followed by the D2H of the 2^L strided runs of y it wrote
// (out row m + Q ii, r_d = 1) while the next chunk computes.
qtt_status_t apply_host_pipelined(qtt_plan* h, const double* x_host, double* y_host, cudaStream_t st) {
  const int ns = int(h->stages.size());
  constexpr int kChunks = 8;
  unsigned char* base = static_cast<unsigned char*>(h->ws);
  int* counters = reinterpret_cast<int*>(base);
  const size_t bb = ws_buf_bytes(h, 1);
  double* buf[2] = {reinterpret_cast<double*>(base + kWsHeader), reinterpret_cast<double*>(base + kWsHeader + bb)};
  if (!h->copy_stream && cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
    return QTT_ERROR_CUDA;
  if (h->pipe_events.empty()) {
    h->pipe_events.resize(2 * kChunks + 2);
    for (auto& ev : h->pipe_events)
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return QTT_ERROR_CUDA;
  }
  static const bool no_flags = std::getenv("QTT_NO_COPY_FLAGS") != nullptr;
  if (!no_flags && h->stages.front().plan.variant == qtt::kWide && h->stages.back().plan.variant == qtt::kWide &&
      stream_mem_ops().write && (h->N >> (h->stages.front().plan.k1 - h->stages.front().plan.k0 + 1)) >= 64 &&
      (h->N >> (h->stages.back().plan.k1 - h->stages.back().plan.k0 + 1)) >= 64)
    return apply_host_flagged(h, x_host, y_host, st);
  cudaStream_t cs = h->copy_stream;
  cudaEvent_t* ev = h->pipe_events.data();
  cudaError_t e = cudaEventRecord(ev[2 * kChunks], st);               // copies start after prior work on st
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[2 * kChunks], 0);
  if (e == cudaSuccess) e = cudaMemsetAsync(counters, 0, kWsHeader, st);
  if (e != cudaSuccess) return from_cuda(e);
  auto chunk_rows = [](int64_t M, int c) {
    const int64_t step = (M / kChunks + 63) / 64 * 64;
    return std::min<int64_t>(M, step * c);
  };
  int ctr = ns;   // counters [0, ns) for unchunked stages, then one per chunk
  const double* in = h->hx;
  for (int si = 0; si < ns; ++si) {
    const Stage& S = h->stages[si];
    const int L = S.plan.k1 - S.plan.k0 + 1;
    const int64_t M = int64_t(1) << (h->d - L);
    double* out = (si == ns - 1) ? h->hy : buf[si & 1];
    if (si == 0 || si == ns - 1) {
      for (int c = 0; c < kChunks; ++c) {
        const int64_t m0 = chunk_rows(M, c), m1 = chunk_rows(M, c + 1);
        if (m1 <= m0) continue;
        if (si == 0) {   // x slice [m0 * 2^L, m1 * 2^L) (r_0 = 1)
          const size_t off = size_t(m0) << L, cnt = size_t(m1 - m0) << L;
          e = cudaMemcpyAsync(h->hx + off, x_host + off, cnt * sizeof(double), cudaMemcpyHostToDevice, cs);
          if (e == cudaSuccess) e = cudaEventRecord(ev[c], cs);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[c], 0);
          if (e != cudaSuccess) return from_cuda(e);
        }
        e = launch_stage(h, S, false, in, out, m1 - m0, m0, counters + (ctr++), st);
        if (e != cudaSuccess) return from_cuda(e);
        if (si == ns - 1) {   // y rows m0..m1 of every output block ii (r_d = 1)
          e = cudaEventRecord(ev[kChunks + c], st);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[kChunks + c], 0);
          if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(y_host + m0, size_t(M) * sizeof(double), h->hy + m0, size_t(M) * sizeof(double),
                                  size_t(m1 - m0) * sizeof(double), size_t(1) << L, cudaMemcpyDeviceToHost, cs);
          if (e != cudaSuccess) return from_cuda(e);
        }
      }
    } else {
      e = launch_stage(h, S, false, in, out, M, 0, counters + si, st);
      if (e != cudaSuccess) return from_cuda(e);
    }
    in = out;
  }
  e = cudaEventRecord(ev[2 * kChunks + 1], cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[2 * kChunks + 1], 0);
  if (e == cudaSuccess) e = cudaEventRecord(h->last, st);
  return from_cuda(e);
}

// enqueue() through a cached CUDA graph: captured once per (x, y, ws, nrhs) on
// an internal stream, then replayed on `st` with one launch.  Falls back to a
// plain enqueue while stage timing is on, when `st` is itself being captured,
// or with QTT_NO_GRAPH set.
qtt_status_t enqueue_graphed(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st) {
  static const bool no_graph = std::getenv("QTT_NO_GRAPH") != nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (no_graph || h->timing || cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return enqueue(h, x, y, nrhs, ws, st);
  }
  for (auto& g : h->graphs)
    if (g.x == x && g.y == y && g.ws == ws && g.nrhs == nrhs) {
      cudaError_t e = cudaGraphLaunch(g.exec, st);
      if (e == cudaSuccess) e = cudaEventRecord(h->last, st);
      return from_cuda(e);
    }
  if (!h->capture_stream && cudaStreamCreateWithFlags(&h->capture_stream, cudaStreamNonBlocking) != cudaSuccess)
    return QTT_ERROR_CUDA;
  cudaError_t e = cudaStreamBeginCapture(h->capture_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return from_cuda(e);
  const qtt_status_t s = enqueue(h, x, y, nrhs, ws, h->capture_stream);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(h->capture_stream, &graph);
  if (s != QTT_SUCCESS) {
    if (graph) cudaGraphDestroy(graph);
    return s;
  }
  if (e != cudaSuccess) return from_cuda(e);
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return from_cuda(e);
  if (h->graphs.size() >= 8) {
    cudaGraphExecDestroy(h->graphs.front().exec);
    h->graphs.erase(h->graphs.begin());
  }
  h->graphs.push_back({x, y, ws, nrhs, exec});
  e = cudaGraphLaunch(exec, st);
  if (e == cudaSuccess) e = cudaEventRecord(h->last, st);
  return from_cuda(e);
}

// The cached workspace is shared by every apply on the handle: order this one
// after the previous one when that was enqueued on another stream (skipped
// while `st` is being captured by the caller).
qtt_status_t order_after_last(qtt_plan* h, cudaStream_t st) {
  if (!h->has_last || h->last_stream == st) return QTT_SUCCESS;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return QTT_SUCCESS;
  }
  return from_cuda(cudaStreamWaitEvent(st, h->last, 0));
}

qtt_status_t check_apply_args(qtt_plan* h, const double* x, const double* y, int64_t nrhs) {
  if (!h || !x || !y || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  if (h->shard_bits) return QTT_ERROR_INVALID_VALUE;   // shard handles use qtt_shard_apply
  // N * nrhs <= 2^31 keeps every GEMM row index a valid 32-bit TMA coordinate
  if (nrhs > (int64_t(1) << 31) / h->N) return QTT_ERROR_NOT_SUPPORTED;
  const uintptr_t xs = reinterpret_cast<uintptr_t>(x), ys = reinterpret_cast<uintptr_t>(y);
  const uintptr_t bytes = uintptr_t(h->N) * uintptr_t(nrhs) * sizeof(double);
  if (xs < ys + bytes && ys < xs + bytes) return QTT_ERROR_INVALID_VALUE;
  if ((xs % 16) || (ys % 16)) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(x, h->device) || !is_device_ptr(y, h->device)) return QTT_ERROR_NOT_SUPPORTED;
  return QTT_SUCCESS;
}

}  // namespace

extern "C" {

const char* qtt_status_string(qtt_status_t s) {
  switch (s) {
    case QTT_SUCCESS: return "QTT_SUCCESS";
    case QTT_ERROR_INVALID_VALUE: return "QTT_ERROR_INVALID_VALUE";
    case QTT_ERROR_NOT_SUPPORTED: return "QTT_ERROR_NOT_SUPPORTED";
    case QTT_ERROR_OUT_OF_MEMORY: return "QTT_ERROR_OUT_OF_MEMORY";
    case QTT_ERROR_CUDA: return "QTT_ERROR_CUDA";
  }
  return "QTT_ERROR_UNKNOWN";
}

qtt_status_t qtt_create(qtt_handle_t* out, int d, const int64_t* ranks, const double* const* cores) {
  return qtt_create_ex(out, d, ranks, cores, qtt::kMaxStageLevels);
}

static qtt_status_t create_impl(qtt_handle_t* out, int d, const int64_t* ranks, const double* const* cores,
                                int max_stage_levels, int shard_bits, int shard_part) {
  const int64_t* const full_ranks = ranks;
  const double* const* const full_cores = cores;
  if (!out) return QTT_ERROR_INVALID_VALUE;
  *out = nullptr;
  if (d < 1 || d > 30 || !ranks || !cores || max_stage_levels < 1) return QTT_ERROR_INVALID_VALUE;
  if (ranks[0] != 1 || ranks[d] != 1) return QTT_ERROR_INVALID_VALUE;
  for (int k = 0; k <= d; ++k)
    if (ranks[k] < 1 || ranks[k] > 4096) return QTT_ERROR_INVALID_VALUE;
  for (int k = 0; k < d; ++k)
    if (!cores[k]) return QTT_ERROR_INVALID_VALUE;
  if (shard_bits < 0 || shard_bits >= d || shard_part < 0 || shard_part >= (1 << shard_bits))
    return QTT_ERROR_INVALID_VALUE;
  qtt_plan* h = nullptr;
  try {
    h = new qtt_plan();
  } catch (const std::bad_alloc&) {
    return QTT_ERROR_OUT_OF_MEMORY;
  }
  if (cudaGetDevice(&h->device) != cudaSuccess) {
    cudaGetLastError();
    delete h;
    return QTT_ERROR_NOT_SUPPORTED;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, h->device) != cudaSuccess) {
    delete h;
    return QTT_ERROR_CUDA;
  }
  if (prop.major != 10 || prop.minor != 0) {
    delete h;
    return QTT_ERROR_NOT_SUPPORTED;   // built for sm_100a only
  }
  h->num_sms = prop.multiProcessorCount;
  h->smem_optin = prop.sharedMemPerBlockOptin;
  // a shard applies the local levels 1..d-s; the rest is its projection
  const int dl = d - shard_bits;
  h->shard_bits = shard_bits;
  h->shard_part = shard_part;
  h->d = dl;
  h->N = int64_t(1) << dl;
  h->ranks.assign(ranks, ranks + dl + 1);
  // A shard's local output T has rows of r_{d-s} doubles that the projection
  // reads with 16-byte vector / TMA accesses: an odd r_{d-s} is padded by one
  // zero bond column (an extra output of core d-s that is identically 0).
  std::vector<const double*> lcores(cores, cores + d);
  std::vector<double> padded;
  if (shard_bits && (ranks[dl] % 2)) {
    const int ra = int(ranks[dl - 1]), rb = int(ranks[dl]);
    padded.assign(size_t(ra) * 4 * (rb + 1), 0.0);
    for (size_t q = 0; q < size_t(ra) * 4; ++q)
      std::copy(cores[dl - 1] + q * rb, cores[dl - 1] + (q + 1) * rb, padded.begin() + q * (rb + 1));
    lcores[dl - 1] = padded.data();
    h->ranks[dl] = rb + 1;
  }
  cores = lcores.data();
  ranks = h->ranks.data();
  qtt_status_t st = QTT_SUCCESS;
  try {
    const std::vector<qtt::StagePlan> plan = qtt::plan_stages(dl, ranks, h->smem_optin, max_stage_levels);
    h->stages.resize(plan.size());
    for (size_t s = 0; s < plan.size(); ++s) {
      h->stages[s].plan = plan[s];
      // the intermediate buffers hold only stage-boundary ranks (and a shard's local output)
      if (s + 1 < plan.size() || shard_bits)
        h->max_interior_rank = std::max<int64_t>(h->max_interior_rank, plan[s].r_out);
    }
    for (size_t s = 0; s < plan.size() && st == QTT_SUCCESS; ++s) st = upload_stage(h, h->stages[s], cores);
    if (st == QTT_SUCCESS && shard_bits) {
      qtt::StagePlan& pp = h->proj.plan;
      const int rp = int(h->ranks[dl]), P = 1 << shard_bits;   // padded local top rank
      const int r = int(full_ranks[dl]);
      if (!qtt::projection_plan(rp, shard_bits, h->smem_optin, &pp)) {
        st = QTT_ERROR_NOT_SUPPORTED;
      } else {
        const std::vector<double> Wp = shard_projection(d, full_ranks, full_cores, shard_bits, shard_part);
        std::vector<double> pk;
        cudaError_t e;
        if (pp.variant == qtt::kWide) {
          e = qtt::wide_prepare(pp.NB, h->smem_optin);
          h->proj.ctas_per_sm = 1;
          pk = pack_wide_fn(pp, [&](int kk, int n) { return (kk < r && n < P) ? Wp[size_t(n) * r + kk] : 0.0; });
        } else {
          e = qtt::dmma_prepare(pp.KB, pp.NB, h->smem_optin);
          int occ = 0;
          if (e == cudaSuccess) e = qtt::dmma_occupancy(pp.KB, pp.NB, pp.smem, &occ);
          h->proj.ctas_per_sm = std::max(1, occ);
          pk = pack_dmma_fn(pp, [&](int kk, int n) {
            return (kk < r && n / 2 < P && n % 2 == 0) ? Wp[size_t(n / 2) * r + kk] : 0.0;
          });
        }
        if (e == cudaSuccess) e = cudaMalloc(&h->proj.d_bpack, pk.size() * sizeof(double));
        if (e == cudaSuccess)
          e = cudaMemcpy(h->proj.d_bpack, pk.data(), pk.size() * sizeof(double), cudaMemcpyHostToDevice);
        st = from_cuda(e);
      }
    }
    h->d_raw.assign(dl, nullptr);
    for (int k = 0; k < dl && st == QTT_SUCCESS; ++k) {
      const size_t bytes = size_t(ranks[k]) * 4 * ranks[k + 1] * sizeof(double);
      cudaError_t e = cudaMalloc(&h->d_raw[k], bytes);
      if (e == cudaSuccess) e = cudaMemcpy(h->d_raw[k], cores[k], bytes, cudaMemcpyHostToDevice);
      st = from_cuda(e);
    }
  } catch (const std::bad_alloc&) {
    st = QTT_ERROR_OUT_OF_MEMORY;
  }
  if (st == QTT_SUCCESS && cudaEventCreateWithFlags(&h->last, cudaEventDisableTiming) != cudaSuccess)
    st = QTT_ERROR_CUDA;
  if (st == QTT_SUCCESS && cudaDeviceSynchronize() != cudaSuccess) st = QTT_ERROR_CUDA;
  if (st != QTT_SUCCESS) {
    free_plan(h);
    return st;
  }
  h->stage_ms.assign(h->stages.size(), 0.0);
  *out = h;
  return QTT_SUCCESS;
}

qtt_status_t qtt_create_ex(qtt_handle_t* out, int d, const int64_t* ranks, const double* const* cores,
                           int max_stage_levels) {
  return create_impl(out, d, ranks, cores, max_stage_levels, 0, 0);
}

qtt_status_t qtt_create_shard(qtt_handle_t* out, int d, const int64_t* ranks, const double* const* cores,
                              int log2_parts, int part) {
  if (log2_parts < 1) return QTT_ERROR_INVALID_VALUE;
  return create_impl(out, d, ranks, cores, qtt::kMaxStageLevels, log2_parts, part);
}

static qtt_status_t check_shard_args(qtt_plan* h, const double* x, const double* send, int64_t nrhs) {
  if (!h || !x || !send || nrhs < 1 || h->shard_bits == 0) return QTT_ERROR_INVALID_VALUE;
  if (nrhs > (int64_t(1) << 31) / (h->N << h->shard_bits)) return QTT_ERROR_NOT_SUPPORTED;
  const uintptr_t xs = reinterpret_cast<uintptr_t>(x), ys = reinterpret_cast<uintptr_t>(send);
  const uintptr_t xb = uintptr_t(h->N) * uintptr_t(nrhs) * sizeof(double);
  const uintptr_t yb = xb << h->shard_bits;
  if (xs < ys + yb && ys < xs + xb) return QTT_ERROR_INVALID_VALUE;
  if ((xs % 16) || (ys % 16)) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(x, h->device) || !is_device_ptr(send, h->device)) return QTT_ERROR_NOT_SUPPORTED;
  return QTT_SUCCESS;
}

qtt_status_t qtt_shard_apply_ws(qtt_handle_t h, const double* x_local, double* send, int64_t nrhs, void* ws,
                                size_t ws_bytes, qtt_stream_t stream) {
  qtt_status_t s = check_shard_args(h, x_local, send, nrhs);
  if (s != QTT_SUCCESS) return s;
  if (!ws || ws_bytes < ws_bytes_for(h, nrhs)) return QTT_ERROR_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(ws) % 256) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(ws)) return QTT_ERROR_NOT_SUPPORTED;
  try {
    DeviceGuard g(h->device);
    return enqueue(h, x_local, send, nrhs, ws, reinterpret_cast<cudaStream_t>(stream));
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_shard_apply(qtt_handle_t h, const double* x_local, double* send, int64_t nrhs,
                             qtt_stream_t stream) {
  qtt_status_t s = check_shard_args(h, x_local, send, nrhs);
  if (s != QTT_SUCCESS) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    const size_t need = ws_bytes_for(h, nrhs);
    if (need > h->ws_bytes) {
      if (h->ws) cudaFreeAsync(h->ws, h->ws_stream);
      h->ws = nullptr;
      h->ws_bytes = 0;
      cudaError_t e = cudaMallocAsync(&h->ws, need, st);
      if (e != cudaSuccess) {
        h->ws = nullptr;
        return from_cuda(e);
      }
      h->ws_bytes = need;
      h->ws_stream = st;
    }
    qtt_status_t so = order_after_last(h, st);
    if (so == QTT_SUCCESS) so = enqueue(h, x_local, send, nrhs, h->ws, st);
    if (so == QTT_SUCCESS) {
      h->last_stream = st;
      h->has_last = true;
    }
    return so;
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_shard_projection(int d, const int64_t* ranks, const double* const* cores, int log2_parts,
                                  int part, double* W) {
  if (d < 2 || d > 30 || !ranks || !cores || !W || log2_parts < 1 || log2_parts >= d || part < 0 ||
      part >= (1 << log2_parts))
    return QTT_ERROR_INVALID_VALUE;
  if (ranks[0] != 1 || ranks[d] != 1) return QTT_ERROR_INVALID_VALUE;
  for (int k = 0; k <= d; ++k)
    if (ranks[k] < 1 || ranks[k] > 4096) return QTT_ERROR_INVALID_VALUE;
  for (int k = d - log2_parts; k < d; ++k)
    if (!cores[k]) return QTT_ERROR_INVALID_VALUE;
  try {
    const std::vector<double> Wp = shard_projection(d, ranks, cores, log2_parts, part);
    std::copy(Wp.begin(), Wp.end(), W);
  } catch (...) {
    return QTT_ERROR_OUT_OF_MEMORY;
  }
  return QTT_SUCCESS;
}

qtt_status_t qtt_workspace_size(qtt_handle_t h, int64_t nrhs, size_t* bytes) {
  if (!h || !bytes || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  *bytes = ws_bytes_for(h, nrhs);
  return QTT_SUCCESS;
}

qtt_status_t qtt_apply_ws(qtt_handle_t h, const double* x, double* y, int64_t nrhs, void* ws,
                          size_t ws_bytes, qtt_stream_t stream) {
  qtt_status_t s = check_apply_args(h, x, y, nrhs);
  if (s != QTT_SUCCESS) return s;
  const size_t need = ws_bytes_for(h, nrhs);
  if (!ws || ws_bytes < need) return QTT_ERROR_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(ws) % 256) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(ws)) return QTT_ERROR_NOT_SUPPORTED;
  try {
    DeviceGuard g(h->device);
    return enqueue_graphed(h, x, y, nrhs, ws, reinterpret_cast<cudaStream_t>(stream));
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_apply(qtt_handle_t h, const double* x, double* y, int64_t nrhs, qtt_stream_t stream) {
  qtt_status_t s = check_apply_args(h, x, y, nrhs);
  if (s != QTT_SUCCESS) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    const size_t need = ws_bytes_for(h, nrhs);
    if (need > h->ws_bytes) {
      if (h->ws) {
        // the old buffer may still be in use by work on its stream
        cudaFreeAsync(h->ws, h->ws_stream);
        for (size_t i = h->graphs.size(); i-- > 0;)
          if (h->graphs[i].ws == h->ws) {
            cudaGraphExecDestroy(h->graphs[i].exec);
            h->graphs.erase(h->graphs.begin() + i);
          }
        h->ws = nullptr;
        h->ws_bytes = 0;
      }
      cudaError_t e = cudaMallocAsync(&h->ws, need, st);
      if (e != cudaSuccess) {
        h->ws = nullptr;
        return from_cuda(e);
      }
      h->ws_bytes = need;
      h->ws_stream = st;
    }
    const qtt_status_t so = order_after_last(h, st);
    if (so != QTT_SUCCESS) return so;
    const qtt_status_t s2 = enqueue_graphed(h, x, y, nrhs, h->ws, st);
    if (s2 == QTT_SUCCESS) {
      h->last_stream = st;
      h->has_last = true;
    }
    return s2;
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_apply_host(qtt_handle_t h, const double* x_host, double* y_host, int64_t nrhs,
                            qtt_stream_t stream) {
  if (!h || !x_host || !y_host || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    const size_t elems = size_t(h->N) * size_t(nrhs);
    if (elems > h->h_elems) {
      if (h->hx) cudaFree(h->hx);
      if (h->hy) cudaFree(h->hy);
      h->hx = h->hy = nullptr;
      h->h_elems = 0;
      cudaError_t e = cudaMalloc(&h->hx, elems * sizeof(double));
      if (e == cudaSuccess) e = cudaMalloc(&h->hy, elems * sizeof(double));
      if (e != cudaSuccess) return from_cuda(e);
      h->h_elems = elems;
    }
    // pipelined copies: one RHS, at least two stages, enough rows to chunk
    if (nrhs == 1 && h->stages.size() >= 2 && h->shard_bits == 0 && !h->timing &&
        (h->N >> (h->stages.front().plan.k1 - h->stages.front().plan.k0 + 1)) >= 8 * 64 &&
        (h->N >> (h->stages.back().plan.k1 - h->stages.back().plan.k0 + 1)) >= 8 * 64) {
      const size_t need = ws_bytes_for(h, 1);
      if (need > h->ws_bytes) {
        if (h->ws) cudaFreeAsync(h->ws, h->ws_stream);
        h->ws = nullptr;
        h->ws_bytes = 0;
        for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
        h->graphs.clear();
        cudaError_t e = cudaMallocAsync(&h->ws, need, st);
        if (e != cudaSuccess) {
          h->ws = nullptr;
          return from_cuda(e);
        }
        h->ws_bytes = need;
        h->ws_stream = st;
      }
      qtt_status_t s = order_after_last(h, st);
      if (s == QTT_SUCCESS) s = apply_host_pipelined(h, x_host, y_host, st);
      if (s != QTT_SUCCESS) return s;
      h->last_stream = st;
      h->has_last = true;
      return from_cuda(cudaStreamSynchronize(st));
    }
    cudaError_t e = cudaMemcpyAsync(h->hx, x_host, elems * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return from_cuda(e);
    qtt_status_t s = qtt_apply(h, h->hx, h->hy, nrhs, stream);
    if (s != QTT_SUCCESS) return s;
    e = cudaMemcpyAsync(y_host, h->hy, elems * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return from_cuda(e);
    return from_cuda(cudaStreamSynchronize(st));
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

static qtt_status_t morton_common(const double* in, double* out, int dim, int levels, int64_t nrhs,
                                  qtt_stream_t stream, bool pack) {
  if (!in || !out || dim < 1 || dim > 3 || levels < 1 || dim * levels > 30 || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  const int64_t N = int64_t(1) << (dim * levels);
  if (nrhs > (int64_t(1) << 40) / N) return QTT_ERROR_INVALID_VALUE;
  const uintptr_t a = reinterpret_cast<uintptr_t>(in), b = reinterpret_cast<uintptr_t>(out);
  const uintptr_t bytes = uintptr_t(N) * uintptr_t(nrhs) * sizeof(double);
  if (a < b + bytes && b < a + bytes) return QTT_ERROR_INVALID_VALUE;
  if ((a % 8) || (b % 8)) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(in) || !is_device_ptr(out)) return QTT_ERROR_NOT_SUPPORTED;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return QTT_ERROR_CUDA;
  return from_cuda(qtt::launch_morton(in, out, dim, levels, nrhs, pack, reinterpret_cast<cudaStream_t>(stream), sms));
}

qtt_status_t qtt_morton_pack(const double* grid, double* x, int dim, int levels, int64_t nrhs, qtt_stream_t stream) {
  return morton_common(grid, x, dim, levels, nrhs, stream, true);
}

qtt_status_t qtt_morton_unpack(const double* x, double* grid, int dim, int levels, int64_t nrhs,
                               qtt_stream_t stream) {
  return morton_common(x, grid, dim, levels, nrhs, stream, false);
}

qtt_status_t qtt_apply_grid(qtt_handle_t h, const double* grid_in, double* grid_out, int dim, int64_t nrhs,
                            qtt_stream_t stream) {
  if (!h || !grid_in || !grid_out || dim < 1 || dim > 3 || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  if (h->d % dim) return QTT_ERROR_INVALID_VALUE;
  const int levels = h->d / dim;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    const size_t elems = size_t(h->N) * size_t(nrhs);
    if (elems > h->g_elems) {
      if (h->gx) cudaFreeAsync(h->gx, h->g_stream);
      if (h->gy) cudaFreeAsync(h->gy, h->g_stream);
      h->gx = h->gy = nullptr;
      h->g_elems = 0;
      cudaError_t e = cudaMallocAsync(&h->gx, elems * sizeof(double), st);
      if (e == cudaSuccess) e = cudaMallocAsync(&h->gy, elems * sizeof(double), st);
      if (e != cudaSuccess) return from_cuda(e);
      h->g_elems = elems;
      h->g_stream = st;
    }
    qtt_status_t s = qtt_morton_pack(grid_in, h->gx, dim, levels, nrhs, stream);
    if (s != QTT_SUCCESS) return s;
    s = qtt_apply(h, h->gx, h->gy, nrhs, stream);
    if (s != QTT_SUCCESS) return s;
    return qtt_morton_unpack(h->gy, grid_out, dim, levels, nrhs, stream);
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

// ---------------------------------------------------------------- compressed matvec (NEXT-3)
static qtt_status_t compressed_common(qtt_handle_t h, const int64_t* b_ranks, const double* const* b_cores,
                                      double* c_dense, double* c_cores, size_t c_cores_bytes, int64_t* c_ranks,
                                      qtt_stream_t stream) {
  if (!h || !b_ranks || !b_cores || h->shard_bits) return QTT_ERROR_INVALID_VALUE;
  const int d = h->d;
  if (b_ranks[0] != 1 || b_ranks[d] != 1) return QTT_ERROR_INVALID_VALUE;
  for (int k = 0; k <= d; ++k)
    if (b_ranks[k] < 1 || b_ranks[k] > 4096) return QTT_ERROR_INVALID_VALUE;
  for (int k = 0; k < d; ++k)
    if (!b_cores[k]) return QTT_ERROR_INVALID_VALUE;
  std::vector<int64_t> R(d + 1);
  for (int k = 0; k <= d; ++k) {
    R[k] = h->ranks[k] * b_ranks[k];
    if (R[k] > 4096) return QTT_ERROR_NOT_SUPPORTED;
  }
  if (c_ranks)
    for (int k = 0; k <= d; ++k) c_ranks[k] = R[k];
  std::vector<size_t> coff(d + 1, 0), boff(d + 1, 0);
  for (int k = 0; k < d; ++k) {
    coff[k + 1] = coff[k] + size_t(R[k]) * 2 * R[k + 1];
    boff[k + 1] = boff[k] + size_t(b_ranks[k]) * 2 * b_ranks[k + 1];
  }
  if (c_cores && c_cores_bytes < coff[d] * sizeof(double)) return QTT_ERROR_INVALID_VALUE;
  if (c_dense && !is_device_ptr(c_dense)) return QTT_ERROR_NOT_SUPPORTED;
  if (c_cores && !is_device_ptr(c_cores)) return QTT_ERROR_NOT_SUPPORTED;
  if (c_dense && (reinterpret_cast<uintptr_t>(c_dense) % 16)) return QTT_ERROR_NOT_SUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    // b's cores: host -> device (pageable copy, synchronous w.r.t. the host arrays)
    double* dV = nullptr;
    cudaError_t e = cudaMallocAsync(&dV, std::max<size_t>(boff[d], 1) * sizeof(double), st);
    if (e != cudaSuccess) return from_cuda(e);
    for (int k = 0; k < d && e == cudaSuccess; ++k)
      e = cudaMemcpyAsync(dV + boff[k], b_cores[k], (boff[k + 1] - boff[k]) * sizeof(double),
                          cudaMemcpyHostToDevice, st);
    double* dC = c_cores;
    if (e == cudaSuccess && !dC) e = cudaMallocAsync(&dC, coff[d] * sizeof(double), st);
    void* ws = nullptr;
    const size_t wsb = c_dense ? qtt::densify_workspace_bytes(d, R.data()) : 0;
    if (e == cudaSuccess && wsb) e = cudaMallocAsync(&ws, wsb, st);
    if (e == cudaSuccess) {
      std::vector<const double*> G(h->d_raw.begin(), h->d_raw.end()), V(d);
      std::vector<double*> C(d);
      for (int k = 0; k < d; ++k) {
        V[k] = dV + boff[k];
        C[k] = dC + coff[k];
      }
      e = qtt::compressed_cores(d, h->ranks.data(), G.data(), b_ranks, V.data(), C.data(), st, h->num_sms);
      if (e == cudaSuccess && c_dense) {
        std::vector<const double*> Cc(C.begin(), C.end());
        e = qtt::tt_densify(d, R.data(), Cc.data(), c_dense, ws, st, h->num_sms, h->smem_optin);
      }
    }
    if (ws) cudaFreeAsync(ws, st);
    if (dC && dC != c_cores) cudaFreeAsync(dC, st);
    cudaFreeAsync(dV, st);
    // the host core arrays may be freed by the caller on return
    cudaError_t se = cudaStreamSynchronize(st);
    return from_cuda(e != cudaSuccess ? e : se);
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_compressed_matvec(qtt_handle_t h, const int64_t* b_ranks, const double* const* b_cores,
                                   double* c, int64_t* c_ranks, qtt_stream_t stream) {
  if (!c) return QTT_ERROR_INVALID_VALUE;
  return compressed_common(h, b_ranks, b_cores, c, nullptr, 0, c_ranks, stream);
}

qtt_status_t qtt_compressed_matvec_cores(qtt_handle_t h, const int64_t* b_ranks, const double* const* b_cores,
                                         double* c_cores, size_t c_cores_bytes, int64_t* c_ranks,
                                         qtt_stream_t stream) {
  if (!c_cores) return QTT_ERROR_INVALID_VALUE;
  return compressed_common(h, b_ranks, b_cores, nullptr, c_cores, c_cores_bytes, c_ranks, stream);
}

// ---------------------------------------------------------------- products (NEXT-1)
static size_t product_vec_bytes(const qtt_product* p, int64_t nrhs) {
  return (size_t(p->N) * size_t(nrhs) * sizeof(double) + 255) / 256 * 256;
}

static size_t product_ws_bytes(const qtt_product* p, int64_t nrhs) {
  size_t f = 0;
  for (auto* h : p->factors) f = std::max(f, ws_bytes_for(h, nrhs));
  const size_t nvec = p->factors.size() >= 3 ? 2 : (p->factors.size() == 2 ? 1 : 0);
  return f + nvec * product_vec_bytes(p, nrhs);
}

qtt_status_t qtt_product_create(qtt_product_t* out, int n_factors, const qtt_handle_t* factors) {
  if (!out) return QTT_ERROR_INVALID_VALUE;
  *out = nullptr;
  if (n_factors < 1 || !factors) return QTT_ERROR_INVALID_VALUE;
  for (int i = 0; i < n_factors; ++i) {
    if (!factors[i]) return QTT_ERROR_INVALID_VALUE;
    if (factors[i]->d != factors[0]->d || factors[i]->device != factors[0]->device) return QTT_ERROR_INVALID_VALUE;
  }
  try {
    qtt_product* p = new qtt_product();
    p->factors.assign(factors, factors + n_factors);
    p->device = factors[0]->device;
    p->N = factors[0]->N;
    *out = p;
  } catch (const std::bad_alloc&) {
    return QTT_ERROR_OUT_OF_MEMORY;
  }
  return QTT_SUCCESS;
}

qtt_status_t qtt_product_workspace_size(qtt_product_t p, int64_t nrhs, size_t* bytes) {
  if (!p || !bytes || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  *bytes = product_ws_bytes(p, nrhs);
  return QTT_SUCCESS;
}

qtt_status_t qtt_product_apply_ws(qtt_product_t p, const double* x, double* y, int64_t nrhs, void* ws,
                                  size_t ws_bytes, qtt_stream_t stream) {
  if (!p) return QTT_ERROR_INVALID_VALUE;
  qtt_status_t s = check_apply_args(p->factors[0], x, y, nrhs);
  if (s != QTT_SUCCESS) return s;
  const size_t need = product_ws_bytes(p, nrhs);
  if (!ws || ws_bytes < need) return QTT_ERROR_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(ws) % 256) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(ws)) return QTT_ERROR_NOT_SUPPORTED;
  try {
    DeviceGuard g(p->device);
    const int n = int(p->factors.size());
    unsigned char* base = static_cast<unsigned char*>(ws);
    const size_t vb = product_vec_bytes(p, nrhs);
    double* tmp[2] = {reinterpret_cast<double*>(base), reinterpret_cast<double*>(base + vb)};
    const size_t nvec = n >= 3 ? 2 : (n == 2 ? 1 : 0);
    void* fws = base + nvec * vb;
    const double* in = x;
    // F_{n-1} first; each factor's stages read the previous factor's output
    for (int i = n - 1, step = 0; i >= 0; --i, ++step) {
      double* out = (i == 0) ? y : tmp[step & 1];
      s = enqueue(p->factors[i], in, out, nrhs, fws, reinterpret_cast<cudaStream_t>(stream));
      if (s != QTT_SUCCESS) return s;
      in = out;
    }
    return QTT_SUCCESS;
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_product_apply(qtt_product_t p, const double* x, double* y, int64_t nrhs, qtt_stream_t stream) {
  if (!p) return QTT_ERROR_INVALID_VALUE;
  qtt_status_t s = check_apply_args(p->factors[0], x, y, nrhs);
  if (s != QTT_SUCCESS) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(p->device);
    const size_t need = product_ws_bytes(p, nrhs);
    if (need > p->ws_bytes) {
      if (p->ws) cudaFreeAsync(p->ws, p->ws_stream);
      p->ws = nullptr;
      p->ws_bytes = 0;
      cudaError_t e = cudaMallocAsync(&p->ws, need, st);
      if (e != cudaSuccess) {
        p->ws = nullptr;
        return from_cuda(e);
      }
      p->ws_bytes = need;
      p->ws_stream = st;
    }
    return qtt_product_apply_ws(p, x, y, nrhs, p->ws, p->ws_bytes, stream);
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_product_destroy(qtt_product_t p) {
  if (!p) return QTT_SUCCESS;
  DeviceGuard g(p->device);
  if (p->ws) {
    if (p->ws_stream) cudaStreamSynchronize(p->ws_stream);
    cudaFree(p->ws);
  }
  delete p;
  return QTT_SUCCESS;
}

qtt_status_t qtt_get_info(qtt_handle_t h, int* d, int64_t* N, int64_t* max_rank, double* flops_per_rhs,
                          int* launches_per_apply) {
  if (!h) return QTT_ERROR_INVALID_VALUE;
  if (d) *d = h->d;
  if (N) *N = h->N;
  if (max_rank) *max_rank = *std::max_element(h->ranks.begin(), h->ranks.end());
  if (flops_per_rhs) {
    double s = 0;
    for (int k = 0; k < h->d; ++k) s += double(h->ranks[k]) * double(h->ranks[k + 1]);
    *flops_per_rhs = 4.0 * s * double(h->N);
  }
  if (launches_per_apply) *launches_per_apply = int(h->stages.size()) + (h->shard_bits ? 1 : 0);
  return QTT_SUCCESS;
}

qtt_status_t qtt_get_stage(qtt_handle_t h, int s, int* k_first, int* k_last, int* variant) {
  if (h && h->shard_bits && s == int(h->stages.size())) {   // a shard's projection launch
    if (k_first) *k_first = h->d + 1;
    if (k_last) *k_last = h->d + h->shard_bits;
    if (variant) *variant = h->proj.plan.variant;
    return QTT_SUCCESS;
  }
  if (!h || s < 0 || s >= int(h->stages.size())) return QTT_ERROR_INVALID_VALUE;
  if (k_first) *k_first = h->stages[s].plan.k0;
  if (k_last) *k_last = h->stages[s].plan.k1;
  if (variant) *variant = h->stages[s].plan.variant;
  return QTT_SUCCESS;
}

qtt_status_t qtt_set_stage_timing(qtt_handle_t h, int enable) {
  if (!h) return QTT_ERROR_INVALID_VALUE;
  h->timing = enable != 0;
  return QTT_SUCCESS;
}

qtt_status_t qtt_stage_times(qtt_handle_t h, float* ms, int n_stages, int* n_applies) {
  if (!h) return QTT_ERROR_INVALID_VALUE;
  DeviceGuard g(h->device);
  qtt_status_t st = QTT_SUCCESS;
  for (auto& e : h->pending) {
    float t = 0;
    if (cudaEventSynchronize(e.stop) != cudaSuccess || cudaEventElapsedTime(&t, e.start, e.stop) != cudaSuccess)
      st = QTT_ERROR_CUDA;
    h->stage_ms[e.stage] += t;
    cudaEventDestroy(e.start);
    cudaEventDestroy(e.stop);
  }
  h->pending.clear();
  if (ms)
    for (int s = 0; s < n_stages && s < int(h->stages.size()); ++s) ms[s] = float(h->stage_ms[s]);
  if (n_applies) *n_applies = h->timed_applies;
  std::fill(h->stage_ms.begin(), h->stage_ms.end(), 0.0);
  h->timed_applies = 0;
  return st;
}

qtt_status_t qtt_destroy(qtt_handle_t h) {
  if (!h) return QTT_SUCCESS;
  DeviceGuard g(h->device);
  if (h->last) cudaEventSynchronize(h->last);
  if (h->ws && h->ws_stream) cudaStreamSynchronize(h->ws_stream);
  if (h->gx && h->g_stream) cudaStreamSynchronize(h->g_stream);
  free_plan(h);
  return QTT_SUCCESS;
}

}  // extern "C"
