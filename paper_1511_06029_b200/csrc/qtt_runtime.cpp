// Runtime of libqtt_b200.so: super-core contraction and B-operand packing
// (SURVEY B1), workspace layout, per-stage launches, the per-apply enqueue and
// its CUDA-graph cache, argument checks.  The arithmetic of PAPER.md Alg. 2
// runs entirely in the kernels; nothing here touches vector data.
#include "qtt_runtime.h"

#include <nvtx3/nvToolsExt.h>   // header-only NVTX: host ranges per stage for nsys / ncu --nvtx

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

namespace qtt {
namespace rt {
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

// Small stage: the same Bmat as the wide stage, in pack_small order.
std::vector<double> pack_small(const double* W, const qtt::StagePlan& sp) {
  const int r_in = sp.r_in, r_out = sp.r_out, n_i = sp.n_i, K = sp.K, nout = sp.n_i * sp.r_out;
  return pack_small_fn(sp, [=](int kk, int n) {
    if (kk >= K || n >= nout) return 0.0;
    const int jj = kk / r_in, a = kk % r_in;
    const int ii = n / r_out, b = n % r_out;
    return W[((size_t(a) * n_i + ii) * n_i + jj) * r_out + b];
  });
}

std::vector<double> pack_fused(const double* W, const qtt::StagePlan& sp) {
  const int r_in = sp.r_in, r_out = sp.r_out, n_i = sp.n_i, K = sp.K, nout = sp.n_i * sp.r_out;
  return pack_fused_fn(sp, [=](int kk, int n) {
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
bool is_device_ptr(const void* p, int dev) {
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
// (the ping-pong intermediate y_k of Alg. 2 at the stage boundaries)
// [split-K partials of the largest split stage, if any].

size_t ws_buf_bytes(const qtt_plan* h, int64_t nrhs) {
  if (h->stages.size() <= 1 && h->fstages.empty() && h->shard_bits == 0) return 0;
  // a fused grid apply also gathers the input grid into buffer 1 (>= 1 double per element)
  const size_t one = size_t(std::max<int64_t>(h->max_interior_rank, 1)) * size_t(h->N) * size_t(nrhs) * sizeof(double);
  return (one + 255) / 256 * 256;
}

// Split-K of a wide stage (1 = none): the planner's, fixed per plan whatever
// the number of RHS or rows of a launch, so every output element is summed in
// the same order in every path (batch-invariant, chunked host-copy launches
// included).
int stage_ksplit(const qtt_plan*, const Stage& S, int64_t) {
  const qtt::StagePlan& sp = S.plan;
  return sp.variant == qtt::kWide && sp.ksplit > 1 ? sp.ksplit : 1;
}

// split-K scratch of one stage: the partial sums, [tiles][S][consumer warps][slot]
static size_t split_bytes(const qtt_plan* h, const Stage& S, int64_t M) {
  const int ks = stage_ksplit(h, S, M);
  if (ks <= 1) return 0;
  const int64_t tiles = (M + qtt::kDmmaRowsPerSubtile - 1) / qtt::kDmmaRowsPerSubtile * S.plan.ncb;
  const int cw = qtt::wide_consumer_warps(S.plan.NB);
  return size_t(tiles) * ks * cw * qtt::split_slot_doubles(S.plan.NB) * sizeof(double);
}

static size_t ws_split_bytes(const qtt_plan* h, int64_t nrhs) {
  size_t m = 0;
  for (const auto& S : h->stages)
    m = std::max(m, split_bytes(h, S, nrhs * (int64_t(1) << (h->d - (S.plan.k1 - S.plan.k0 + 1)))));
  return m;
}

// Split-K scratch after the two buffers (every slot is written by the split
// launch before its reduce launch reads it: no initialisation needed).
cudaError_t setup_split(const qtt_plan* h, void* ws, int64_t nrhs, cudaStream_t, SplitScratch* out) {
  *out = SplitScratch{};
  if (!ws_split_bytes(h, nrhs)) return cudaSuccess;
  out->partial = reinterpret_cast<double*>(static_cast<unsigned char*>(ws) + kWsHeader + 2 * ws_buf_bytes(h, nrhs));
  return cudaSuccess;
}

size_t ws_bytes_for(const qtt_plan* h, int64_t nrhs) {
  return kWsHeader + 2 * ws_buf_bytes(h, nrhs) + ws_split_bytes(h, nrhs);
}

void free_plan(qtt_plan* h) {
  for (auto* v : {&h->stages, &h->fstages})
    for (auto& S : *v) {
      if (S.d_bpack) cudaFree(S.d_bpack);
      if (S.d_core) cudaFree(S.d_core);
      if (S.d_coloff) cudaFree(S.d_coloff);
    }
  for (double* p : h->d_raw)
    if (p) cudaFree(p);
  if (h->proj.d_bpack) cudaFree(h->proj.d_bpack);
  if (h->proj_fused.d_bpack) cudaFree(h->proj_fused.d_bpack);
  if (h->d_peers) cudaFree(h->d_peers);
  if (h->ws) cudaFree(h->ws);
  if (h->gx) cudaFree(h->gx);        // gy lives in the same allocation
  if (h->cmv) cudaFree(h->cmv);
  if (h->ws_used) cudaEventDestroy(h->ws_used);
  if (h->g_used) cudaEventDestroy(h->g_used);
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
  if (sp.variant == qtt::kDiag) {
    // D[ii][a][b] = (G_k0(:, i_1, i_1, :) ... G_k1(:, i_L, i_L, :))[a][b], ii = sum_l i_l 2^(l-1)
    const int r_in = sp.r_in;
    int rc = int(h->ranks[sp.k0]);
    int n = 2;
    std::vector<double> D(size_t(2) * r_in * rc);     // [ii][a][c]
    {
      const double* G = cores[sp.k0 - 1];
      for (int i = 0; i < 2; ++i)
        for (int a = 0; a < r_in; ++a)
          for (int c = 0; c < rc; ++c) D[(size_t(i) * r_in + a) * rc + c] = G[((size_t(a) * 2 + i) * 2 + i) * rc + c];
    }
    for (int k = sp.k0 + 1; k <= sp.k1; ++k) {
      const double* G = cores[k - 1];
      const int rb = int(h->ranks[k]);
      std::vector<double> V(size_t(2 * n) * r_in * rb, 0.0);
      for (int i = 0; i < 2; ++i)
        for (int ii = 0; ii < n; ++ii)
          for (int a = 0; a < r_in; ++a) {
            double* v = &V[(size_t(ii + n * i) * r_in + a) * rb];
            const double* u = &D[(size_t(ii) * r_in + a) * rc];
            for (int c = 0; c < rc; ++c) {
              const double uc = u[c];
              if (uc == 0.0) continue;
              const double* g = G + ((size_t(c) * 2 + i) * 2 + i) * rb;
              for (int b = 0; b < rb; ++b) v[b] += uc * g[b];
            }
          }
      D.swap(V);
      n *= 2;
      rc = rb;
    }
    cudaError_t e = cudaMalloc(&S.d_core, D.size() * sizeof(double));
    if (e != cudaSuccess) return from_cuda(e);
    return from_cuda(cudaMemcpy(S.d_core, D.data(), D.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (sp.variant == qtt::kSmall || sp.variant == qtt::kFused) {
    S.ctas_per_sm = 1;
    const std::vector<double> W = sp.k0 == sp.k1
                                      ? std::vector<double>(cores[sp.k0 - 1], cores[sp.k0 - 1] + size_t(sp.r_in) * 4 * sp.r_out)
                                      : super_core(cores, h->ranks.data(), sp.k0, sp.k1);
    if (sp.variant == qtt::kFused) {
      cudaError_t e = qtt::fused_prepare();
      if (e != cudaSuccess) return from_cuda(e);
    }
    const std::vector<double> pk = sp.variant == qtt::kFused ? pack_fused(W.data(), sp) : pack_small(W.data(), sp);
    cudaError_t e = cudaMalloc(&S.d_bpack, pk.size() * sizeof(double));
    if (e != cudaSuccess) return from_cuda(e);
    return from_cuda(cudaMemcpy(S.d_bpack, pk.data(), pk.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (sp.variant == qtt::kWide) {
    cudaError_t e = qtt::wide_prepare(sp.NB, h->smem_optin);
    if (e != cudaSuccess) return from_cuda(e);
    S.ctas_per_sm = 1;
    {   // epilogue column offsets: column n = ii r_out + b -> (ii << log2_q) r_out + b
      const int log2_q = h->d - (sp.k1 - sp.k0 + 1);
      const int nout = sp.n_i * sp.r_out;
      std::vector<int64_t> co(static_cast<size_t>(nout));
      for (int n = 0; n < nout; ++n)
        co[size_t(n)] = (int64_t(n / sp.r_out) << log2_q) * sp.r_out + n % sp.r_out;
      e = cudaMalloc(&S.d_coloff, co.size() * sizeof(int64_t));
      if (e != cudaSuccess) return from_cuda(e);
      e = cudaMemcpy(S.d_coloff, co.data(), co.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return from_cuda(e);
    }
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

cudaError_t launch_stage(qtt_plan* h, const Stage& S, bool proj, const double* in, double* out, int64_t M,
                         int64_t m_base, int* counter, cudaStream_t st, const WideHooks* hooks,
                         const SplitScratch* split) {
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
  // rows the stage's output holds from `out` on (a chunk's pointer is pre-offset
  // by m_base rows): the whole output is max(M n_i, N) rows of r_out doubles
  a.out_limit = (std::max<int64_t>(M * sp.n_i, h->N) - m_base) * sp.r_out;
  if (hooks) {
    a.peers = hooks->peers;
    a.peer_offset = hooks->peer_offset;
    a.ready = hooks->ready;
    a.ready_val = hooks->ready_val;
    a.ready_rows = hooks->ready_rows;
    a.done = hooks->done;
    a.done_rows = hooks->done_rows;
  }
  cudaError_t e;
  if (sp.variant == qtt::kWide) {
    int64_t tiles = (a.M + qtt::kDmmaRowsPerSubtile - 1) / qtt::kDmmaRowsPerSubtile * sp.ncb;
    const int ks = proj ? 1 : stage_ksplit(h, S, M);
    if (ks > 1 && !split) return cudaErrorInvalidValue;   // caller must provide the scratch
    if (ks > 1) {
      a.ksplit = ks;
      a.kcps = (sp.nchunks + ks - 1) / ks;
      a.partial = split->partial;
      tiles *= ks;
    }
    a.grid = int(std::min<int64_t>(tiles, int64_t(h->num_sms) * (sp.NB <= 8 ? QTT_WIDE_CTAS : 1)));
    if (!proj) {
      static const bool no_coloff = std::getenv("QTT_WIDE_NO_COLOFF") != nullptr;   // A/B
      a.col_off = no_coloff ? nullptr : S.d_coloff;
      if (tiles < (int64_t(1) << 31)) {   // tile -> (row tile, column block) by multiply-shift
        const uint32_t dv = uint32_t(sp.ncb);
        int l = 0;
        while ((uint32_t(1) << l) < dv) ++l;
        if ((dv & (dv - 1)) == 0) {
          a.ncb_mul = 0;
          a.ncb_shr = l;
        } else {
          a.ncb_mul = uint32_t(((uint64_t(1) << (31 + l)) / dv) + 1);
          a.ncb_shr = l - 1;
        }
      } else {
        a.col_off = nullptr;              // the generic epilogue (64-bit tile indices)
      }
    }
    e = qtt::launch_wide(a, st);
  } else if (sp.variant == qtt::kSmall) {
    e = qtt::launch_small(a, st);
  } else if (sp.variant == qtt::kDiag) {
    e = qtt::launch_diag(a, st, h->num_sms);
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

qtt_status_t enqueue(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st,
                     bool fused) {
  unsigned char* base = static_cast<unsigned char*>(ws);
  int* counters = reinterpret_cast<int*>(base);
  const size_t bb = ws_buf_bytes(h, nrhs);
  double* buf[2] = {reinterpret_cast<double*>(base + kWsHeader), reinterpret_cast<double*>(base + kWsHeader + bb)};
  cudaError_t me = cudaMemsetAsync(counters, 0, kWsHeader, st);
  if (me != cudaSuccess) return from_cuda(me);
  SplitScratch split;
  me = setup_split(h, ws, nrhs, st, &split);
  if (me != cudaSuccess) return from_cuda(me);
  const bool scb = split.partial != nullptr;
  const double* in = x;
  const int nloc = int(h->stages.size());
  const int ns = nloc + (h->shard_bits ? 1 : 0);
  for (int si = 0; si < ns; ++si) {
    const bool proj = si == nloc;                  // shard projection stage
    const Stage& S = proj ? (fused ? h->proj_fused : h->proj) : h->stages[si];
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
    WideHooks fh;
    if (proj && fused) {   // write each output block straight into its part's receive slot
      fh.peers = h->d_peers;
      fh.peer_offset = int64_t(h->shard_part) * M;
    }
    char name[64];
    std::snprintf(name, sizeof(name), "qtt stage %d-%d v%d", proj ? h->d + 1 : S.plan.k0,
                  proj ? h->d + h->shard_bits : S.plan.k1, S.plan.variant);
    nvtxRangePushA(name);
    const cudaError_t e = launch_stage(h, S, proj, in, out, M, 0, counters + si, st, (proj && fused) ? &fh : nullptr,
                                       scb ? &split : nullptr);
    nvtxRangePop();
    if (e != cudaSuccess) return from_cuda(e);
    if (h->timing && !proj) {
      cudaEventRecord(ev.stop, st);
      h->pending.push_back(ev);
    }
    in = out;
  }
  if (h->timing) h->timed_applies++;
  // an event recorded inside a capture (ours or the caller's) cannot order
  // later work outside it: only plain enqueues update the handle's last event
  if (st != h->capture_stream && !stream_is_capturing(st)) cudaEventRecord(h->last, st);
  return QTT_SUCCESS;
}

bool use_fused(const qtt_plan* h, int64_t nrhs) {
  return h->fused_on && !h->fstages.empty() && nrhs <= h->fused_max_nrhs && !h->timing && h->shard_bits == 0;
}

qtt_status_t enqueue_fused(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st,
                           bool zero_bar, int morton_dim) {
  unsigned char* base = static_cast<unsigned char*>(ws);
  const size_t bb = ws_buf_bytes(h, nrhs);
  double* buf[2] = {reinterpret_cast<double*>(base + kWsHeader), reinterpret_cast<double*>(base + kWsHeader + bb)};
  qtt::FusedArgs a;
  a.nstages = int(h->fstages.size());
  a.bar = reinterpret_cast<unsigned*>(base + qtt::kFusedBarOffset);
  int64_t max_wt = 1;
  const double* in = x;
  for (int s = 0; s < a.nstages; ++s) {
    const qtt::StagePlan& sp = h->fstages[s].plan;
    qtt::FusedStage& f = a.st[s];
    const int L = sp.k1 - sp.k0 + 1;
    const bool last = s + 1 == a.nstages;
    f.in = in;
    f.out = last ? y : buf[s & 1];
    f.bpack = h->fstages[s].d_bpack;
    f.M = nrhs * (h->N >> L);
    f.out_limit = int64_t(h->N) * nrhs * sp.r_out;
    f.log2_q = h->d - L;
    f.n_i = sp.n_i;
    f.r_out = sp.r_out;
    f.nout = sp.n_i * sp.r_out;
    f.K = sp.K;
    f.nchunks = sp.nchunks;
    f.ncb = sp.ncb;
    f.ks = std::max(1, sp.ksplit);
    f.log2n = h->d;
    // work decomposition, precomputed (the kernel only multiplies and shifts)
    f.mtiles = int((f.M + qtt::kSmallRows - 1) / qtt::kSmallRows);
    {
      const int slots = qtt::kFusedWarps / f.ks;
      f.rgroups = (f.mtiles + slots - 1) / slots;
      f.units = f.rgroups * f.ncb;
      const uint32_t dv = uint32_t(f.rgroups);
      int l = 0;
      while ((uint32_t(1) << l) < dv) ++l;
      if ((dv & (dv - 1)) == 0) {          // a power of two: a shift
        f.rg_mul = 0;
        f.rg_shr = l;
      } else {                             // round-up magic number, exact for u < 2^31
        f.rg_mul = uint32_t(((uint64_t(1) << (31 + l)) / dv) + 1);
        f.rg_shr = l - 1;
      }
      f.cps = (f.nchunks + f.ks - 1) / f.ks;
      f.lks = f.ks >= 8 ? 3 : f.ks >= 4 ? 2 : f.ks >= 2 ? 1 : 0;
      int lr = 0;
      while ((1 << lr) < sp.r_out) ++lr;
      f.lr = lr;
    }
    f.mout_dim = last ? morton_dim : 0;      // the scatter is the last stage's epilogue
    static const bool no_runs = std::getenv("QTT_FUSED_NO_RUNS") != nullptr;   // A/B
    // (a Morton-scattering last stage has r_out = 1: a piece is two consecutive
    // QTT indices x0 = 0, 1, i.e. two adjacent grid points: one 16-byte store)
    f.runs = !no_runs && (f.mout_dim == 0 || sp.r_out == 1) && sp.r_out <= 32 && (32 % sp.r_out) == 0 &&
                     f.log2_q >= 4
                 ? 1
                 : 0;
    // fused grid apply: stage 0 gathers the natural-order grid in its A loads
    // (QTT_FUSED_PREPASS=1: a gather pass into buffer 1 and a grid barrier, A/B)
    // (the gather in the loads recomputes a Morton index per 16-byte load of
    // every unit: cheaper than the pass + barrier only for small grids --
    // c1 9.5 vs 10.3 us, c2 29.6 vs 27.6 us)
    static const bool prepass_env = std::getenv("QTT_FUSED_PREPASS") != nullptr;
    const bool prepass = prepass_env || int64_t(h->N) * nrhs > 8192;
    if (s == 0 && morton_dim && prepass) f.in = buf[1];
    f.in_dim = (s == 0 && morton_dim && !prepass) ? morton_dim : 0;
    a.smem = std::max<size_t>(a.smem, size_t(sp.nchunks) * 128 * 16);
    max_wt = std::max<int64_t>(max_wt, (f.M + qtt::kSmallRows - 1) / qtt::kSmallRows * f.ncb * f.ks);
    in = f.out;
  }
  if (morton_dim && a.st[0].in_dim == 0) {   // stage 0 reads the gathered copy in buffer 1 (after a barrier)
    a.pre_src = x;
    a.pre_dst = buf[1];
    a.pre_dim = morton_dim;
    a.pre_log2n = h->d;
    a.pre_total = int64_t(h->N) * nrhs;
  }
  // enough CTAs for the widest stage's (tile, k-part) warps, at most one per SM
  const int grid = int(std::min<int64_t>(h->num_sms, (max_wt + qtt::kFusedWarps - 1) / qtt::kFusedWarps));
  const bool capturing = stream_is_capturing(st);
  if (zero_bar && capturing) {   // inside a graph: a memset node
    const cudaError_t e = cudaMemsetAsync(a.bar, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return from_cuda(e);
  } else if (zero_bar) {   // a stream memory op (no kernel) clears the arrival counter
    using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    static const WriteValueFn wv = [] {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        f = nullptr;
      cudaGetLastError();
      return reinterpret_cast<WriteValueFn>(f);
    }();
    if (!wv || wv(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(a.bar), 0, 0) != CUDA_SUCCESS) {
      const cudaError_t e = cudaMemsetAsync(a.bar, 0, sizeof(unsigned), st);
      if (e != cudaSuccess) return from_cuda(e);
    }
  }
  // diagnostic: QTT_FUSED_PROFILE=1 times every stage and barrier inside the
  // launch (per CTA %globaltimer) and prints min/max over CTAs to stderr
  static const bool fprof = std::getenv("QTT_FUSED_PROFILE") != nullptr;
  static unsigned long long* d_prof = nullptr;
  if (fprof && !d_prof &&
      cudaMalloc(&d_prof, size_t(h->num_sms) * qtt::kFusedProfSlots * sizeof(unsigned long long)) != cudaSuccess)
    d_prof = nullptr;
  if (fprof && !capturing && d_prof) {
    a.prof = d_prof;
    cudaMemsetAsync(d_prof, 0, size_t(h->num_sms) * qtt::kFusedProfSlots * sizeof(unsigned long long), st);
  }
  static const int frep = std::getenv("QTT_FUSED_REPEAT") ? std::atoi(std::getenv("QTT_FUSED_REPEAT")) : 1;
  a.repeat = std::max(1, frep);
  static const bool no_trigger = std::getenv("QTT_FUSED_NO_TRIGGER") != nullptr;
  a.early_trigger = no_trigger ? 0 : 1;
  nvtxRangePushA("qtt fused apply");
  static const bool graph_nopdl = std::getenv("QTT_FUSED_GRAPH_NOPDL") != nullptr;   // A/B
  cudaError_t e = qtt::launch_fused(a, grid, st, !(graph_nopdl && st == h->capture_stream));
  nvtxRangePop();
  if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorLaunchOutOfResources || e == cudaErrorNotSupported) {
    // the device cannot co-schedule the grid here (e.g. under MPS limits): this
    // handle runs its per-stage plan from now on
    cudaGetLastError();
    if (std::getenv("QTT_DEBUG"))
      std::fprintf(stderr, "qtt: fused launch refused (%s); falling back to the per-stage plan\n",
                   cudaGetErrorString(e));
    h->fused_on = false;
    return morton_dim ? QTT_ERROR_NOT_SUPPORTED : enqueue(h, x, y, nrhs, ws, st);
  }
  if (e == cudaSuccess && a.prof) {
    std::vector<unsigned long long> hp(size_t(grid) * qtt::kFusedProfSlots);
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess)
      e = cudaMemcpy(hp.data(), d_prof, hp.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) {
      unsigned long long t0 = ~0ull;
      for (int b = 0; b < grid; ++b) t0 = std::min(t0, hp[size_t(b) * qtt::kFusedProfSlots]);
      std::fprintf(stderr, "qtt fused profile (grid %d, ns from the first CTA start; min/max over CTAs):", grid);
      for (int slot = 0; slot <= 2 * a.nstages; ++slot) {
        unsigned long long lo = ~0ull, hi = 0;
        for (int b = 0; b < grid; ++b) {
          const unsigned long long v = hp[size_t(b) * qtt::kFusedProfSlots + slot] - t0;
          lo = std::min(lo, v);
          hi = std::max(hi, v);
        }
        std::fprintf(stderr, " %s%d=%llu/%llu", slot == 0 ? "start" : (slot % 2 ? "tiles" : "bar"),
                     slot == 0 ? 0 : (slot - 1) / 2, lo, hi);
      }
      std::fprintf(stderr, "\n  CTA 0, first unit of each stage (ns from its start): ");
      for (int s2 = 0; s2 < a.nstages; ++s2) {
        const unsigned long long* d = &hp[2 * qtt::kFusedMaxStages + 2 + 4 * s2];
        std::fprintf(stderr, " s%d: B-in-smem %lld mma %lld stored %lld;", s2, (long long)(d[1] - d[0]),
                     (long long)(d[2] - d[0]), (long long)(d[3] - d[0]));
      }
      std::fprintf(stderr, "\n");
      // per-warp stamps of the first unit of each stage, CTA 0 and the last CTA
      for (int b : {0, grid - 1})
        for (int s2 = 0; s2 < a.nstages; ++s2) {
          const unsigned long long* d = &hp[size_t(b) * qtt::kFusedProfSlots + 2 * qtt::kFusedMaxStages + 2 + 4 * s2];
          const unsigned long long* w = &hp[size_t(b) * qtt::kFusedProfSlots + qtt::kFusedProfBase +
                                            size_t(s2) * qtt::kFusedWarps * 4];
          std::fprintf(stderr, "  CTA %d s%d (ks %d) warp: A-in / mma / sync / stored (ns from unit start):", b, s2,
                       a.st[s2].ks);
          for (int w2 = 0; w2 < qtt::kFusedWarps; ++w2) {
            auto rel = [&](unsigned long long v) { return v ? (long long)(v - d[0]) : -1ll; };
            std::fprintf(stderr, " [%lld %lld %lld %lld]", rel(w[4 * w2]), rel(w[4 * w2 + 1]), rel(w[4 * w2 + 2]),
                         rel(w[4 * w2 + 3]));
          }
          std::fprintf(stderr, "\n");
        }
    }
  }
  if (e != cudaSuccess) {
    if (std::getenv("QTT_DEBUG"))
      std::fprintf(stderr, "qtt: fused apply (%d stages, grid %d) launch failed: %s\n", a.nstages, grid,
                   cudaGetErrorString(e));
    return from_cuda(e);
  }
  if (!capturing) cudaEventRecord(h->last, st);
  return QTT_SUCCESS;
}

// enqueue() (kind 0) or enqueue_fused() (kind 1, 2 = with the barrier reset)
// through a cached CUDA graph: captured once per (x, y, ws, nrhs, kind) on an
// internal stream, then replayed on `st` with one launch.  A graph launch costs
// the host and the GPU front end less than the cooperative launch it holds
// (DESIGN.md 6.11).  Falls back to a plain enqueue while stage timing is on,
// when `st` is itself being captured, or with QTT_NO_GRAPH set.
qtt_status_t enqueue_graphed(qtt_plan* h, const double* x, double* y, int64_t nrhs, void* ws, cudaStream_t st,
                             int kind) {
  static const bool no_graph = std::getenv("QTT_NO_GRAPH") != nullptr;
  static const bool fused_direct = std::getenv("QTT_FUSED_NO_GRAPH") != nullptr ||
                                   std::getenv("QTT_FUSED_PROFILE") != nullptr;
  static bool capture_broken[3] = {false, false, false};   // the driver refused to capture this kind once
  auto plain = [&](cudaStream_t s2) {
    return kind ? enqueue_fused(h, x, y, nrhs, ws, s2, kind == 2) : enqueue(h, x, y, nrhs, ws, s2);
  };
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (no_graph || h->timing || (kind && (fused_direct || capture_broken[kind])) ||
      cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return plain(st);
  }
  for (auto& g : h->graphs)
    if (g.x == x && g.y == y && g.ws == ws && g.nrhs == nrhs && g.kind == kind) {
      nvtxRangePushA("qtt apply (graph replay)");
      cudaError_t e = cudaGraphLaunch(g.exec, st);
      nvtxRangePop();
      if (e == cudaSuccess) e = cudaEventRecord(h->last, st);
      return from_cuda(e);
    }
  if (!h->capture_stream && cudaStreamCreateWithFlags(&h->capture_stream, cudaStreamNonBlocking) != cudaSuccess)
    return QTT_ERROR_CUDA;
  cudaError_t e = cudaStreamBeginCapture(h->capture_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return from_cuda(e);
  const bool fused_before = h->fused_on;
  const qtt_status_t s = plain(h->capture_stream);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(h->capture_stream, &graph);
  cudaGraphExec_t exec = nullptr;
  if (s == QTT_SUCCESS && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (kind && (s != QTT_SUCCESS || e != cudaSuccess || h->fused_on != fused_before)) {
    // the cooperative launch could not be captured (or fell back to the per-stage
    // plan inside the capture): launch it directly from now on
    if (exec) cudaGraphExecDestroy(exec);
    cudaGetLastError();
    capture_broken[kind] = true;
    h->fused_on = fused_before;
    if (std::getenv("QTT_DEBUG")) std::fprintf(stderr, "qtt: fused launch not capturable; launching directly\n");
    return plain(st);
  }
  if (s != QTT_SUCCESS) return s;
  if (e != cudaSuccess) {
    if (std::getenv("QTT_DEBUG")) std::fprintf(stderr, "qtt: graph capture failed: %s\n", cudaGetErrorString(e));
    return from_cuda(e);
  }
  if (h->graphs.size() >= 8) {
    cudaGraphExecDestroy(h->graphs.front().exec);
    h->graphs.erase(h->graphs.begin());
  }
  h->graphs.push_back({x, y, ws, nrhs, exec, kind});
  e = cudaGraphLaunch(exec, st);
  if (e != cudaSuccess && std::getenv("QTT_DEBUG"))
    std::fprintf(stderr, "qtt: graph launch (kind %d) failed: %s\n", kind, cudaGetErrorString(e));
  if (e == cudaSuccess) e = cudaEventRecord(h->last, st);
  return from_cuda(e);
}

// The cached workspace is shared by every apply on the handle: order this one
// after the previous one when that was enqueued on another stream (skipped
// while `st` is being captured by the caller).
bool stream_is_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

qtt_status_t cached_acquire(void** ptr, size_t* bytes, cudaEvent_t* used, bool pending, size_t need,
                            cudaStream_t st, bool capturing, bool* grew) {
  if (grew) *grew = false;
  if (capturing && need > *bytes) return QTT_ERROR_NOT_SUPPORTED;
  if (!*used && cudaEventCreateWithFlags(used, cudaEventDisableTiming) != cudaSuccess) {
    *used = nullptr;
    return QTT_ERROR_CUDA;
  }
  if (pending && !capturing) {
    const cudaError_t e = cudaStreamWaitEvent(st, *used, 0);
    if (e != cudaSuccess) return from_cuda(e);
  }
  if (need <= *bytes) return QTT_SUCCESS;
  if (*ptr) {
    const cudaError_t e = cudaFreeAsync(*ptr, st);
    if (e != cudaSuccess) return from_cuda(e);
    *ptr = nullptr;
    *bytes = 0;
  }
  if (grew) *grew = true;
  cudaError_t e = cudaMallocAsync(ptr, need, st);
  if (e == cudaErrorMemoryAllocation) {
    // the released block (and other freed blocks) may still sit in the
    // stream-ordered pool, unusable for a larger allocation: wait for the
    // stream, return the pool's free memory to the device and retry once
    cudaGetLastError();
    cudaMemPool_t pool = nullptr;
    int dev = 0;
    if (cudaStreamSynchronize(st) == cudaSuccess && cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(ptr, need, st);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return from_cuda(e);
  }
  *bytes = need;
  return QTT_SUCCESS;
}

qtt_status_t cached_release(cudaEvent_t used, bool* pending, cudaStream_t st, bool capturing) {
  if (capturing || !used) return QTT_SUCCESS;
  const cudaError_t e = cudaEventRecord(used, st);
  if (e != cudaSuccess) return from_cuda(e);
  *pending = true;
  return QTT_SUCCESS;
}

qtt_status_t check_apply_args(qtt_plan* h, const double* x, const double* y, int64_t nrhs) {
  if (!h || !x || !y || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  if (h->shard_bits) return QTT_ERROR_INVALID_VALUE;   // shard handles use qtt_shard_apply
  // an apply's byte range must be addressable (launches are grouped by rhs_group)
  if (nrhs > (int64_t(1) << 60) / h->N) return QTT_ERROR_INVALID_VALUE;
  const uintptr_t xs = reinterpret_cast<uintptr_t>(x), ys = reinterpret_cast<uintptr_t>(y);
  const uintptr_t bytes = uintptr_t(h->N) * uintptr_t(nrhs) * sizeof(double);
  if (xs < ys + bytes && ys < xs + bytes) return QTT_ERROR_INVALID_VALUE;
  if ((xs % 16) || (ys % 16)) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(x, h->device) || !is_device_ptr(y, h->device)) return QTT_ERROR_NOT_SUPPORTED;
  return QTT_SUCCESS;
}

}  // namespace rt
}  // namespace qtt
