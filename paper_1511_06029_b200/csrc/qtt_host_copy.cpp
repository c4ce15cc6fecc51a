// qtt_apply_host with the host<->device copies overlapped with the first and
// last stages (chunked launches, or single launches with device-side copy
// flags when both end stages are wide).
#include "qtt_runtime.h"

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
  SplitScratch split;
  cudaError_t e = cudaMemsetAsync(counters, 0, kWsHeader, st);
  if (e == cudaSuccess) e = setup_split(h, h->ws, 1, st, &split);
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
    e = launch_stage(h, S, false, in, out, M, 0, counters + si, st, (si == 0 || si == ns - 1) ? &hk : nullptr,
                     &split);
    if (e != cudaSuccess) return from_cuda(e);
    in = out;
  }
  // y chunks: rows [m0, m1) of every output block ii, once all their tiles are stored
  const int cw = 4 * qtt::wide_col_groups(SL.plan.NB);        // consumer warps per CTA
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
  SplitScratch split;
  if (e == cudaSuccess) e = setup_split(h, h->ws, 1, st, &split);
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
        e = launch_stage(h, S, false, in, out, m1 - m0, m0, counters + (ctr++), st, nullptr, &split);
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
      e = launch_stage(h, S, false, in, out, M, 0, counters + si, st, nullptr, &split);
      if (e != cudaSuccess) return from_cuda(e);
    }
    in = out;
  }
  e = cudaEventRecord(ev[2 * kChunks + 1], cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[2 * kChunks + 1], 0);
  if (e == cudaSuccess) e = cudaEventRecord(h->last, st);
  return from_cuda(e);
}

}  // namespace rt
}  // namespace qtt
