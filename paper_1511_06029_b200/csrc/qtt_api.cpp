// C ABI of libqtt_b200.so (declared and documented in include/qtt.h): plans,
// applies, shards, introspection and lifetime.  Products, Morton ordering and
// the compressed matvec are in qtt_api_ext.cpp; the runtime they share is
// qtt_runtime.cpp.
#include "qtt_runtime.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

using namespace qtt::rt;

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
    // levels whose cores are diagonal in (i_k, j_k) (exact zeros off the diagonal):
    // block-diagonal digits, planned as streaming diagonal stages
    std::vector<unsigned char> diag(dl, 0);
    for (int k = 0; k < dl; ++k) {
      const double* G = cores[k];
      bool dg = true;
      for (size_t a = 0; a < size_t(ranks[k]) && dg; ++a)
        for (int b = 0; b < ranks[k + 1] && dg; ++b)
          dg = G[(a * 4 + 1) * ranks[k + 1] + b] == 0.0 && G[(a * 4 + 2) * ranks[k + 1] + b] == 0.0;
      diag[k] = dg ? 1 : 0;
    }
    const std::vector<qtt::StagePlan> plan =
        qtt::plan_stages(dl, ranks, h->smem_optin, max_stage_levels, diag.data());
    h->stages.resize(plan.size());
    for (size_t s = 0; s < plan.size(); ++s) {
      h->stages[s].plan = plan[s];
      // the intermediate buffers hold only stage-boundary ranks (and a shard's local output)
      if (s + 1 < plan.size() || shard_bits)
        h->max_interior_rank = std::max<int64_t>(h->max_interior_rank, plan[s].r_out);
    }
    for (size_t s = 0; s < plan.size() && st == QTT_SUCCESS; ++s) st = upload_stage(h, h->stages[s], cores);
    // the fused apply: ONE persistent launch for latency-bound sizes, when the
    // cost model prefers it to the per-stage launches.  Only
    // with the default stage cap (a cap asks for that launch structure).
    static const bool no_fused = std::getenv("QTT_NO_FUSED") != nullptr;
    static const bool force_fused = std::getenv("QTT_FORCE_FUSED") != nullptr;
    if (st == QTT_SUCCESS && !shard_bits && !no_fused && max_stage_levels >= qtt::kMaxStageLevels) {
      double est1 = 0;
      std::vector<qtt::StagePlan> fp = qtt::plan_stages_fused(dl, ranks, max_stage_levels, h->N, &est1);
      int64_t fr = 1;
      for (size_t s = 0; s + 1 < fp.size(); ++s) fr = std::max<int64_t>(fr, fp[s].r_out);
      int64_t pmax = 0;
      for (int64_t p = 1; !fp.empty() && p <= 64; p *= 2) {
        if (2.0 * double(fr) * double(h->N) * double(p) * 8.0 > double(qtt::kFusedMaxL2Bytes)) break;
        // this fused plan at p RHS against the best per-stage plan at p RHS
        double ef = qtt::fused_launch_seconds();
        for (const auto& sp : fp) {
          qtt::StagePlan tmp;
          ef += qtt::fused_stage_seconds(ranks, sp.k0, sp.k1, double(h->N) * double(p), &tmp);
        }
        const std::vector<qtt::StagePlan> rp =
            qtt::plan_stages(dl, ranks, h->smem_optin, max_stage_levels, diag.data(), h->N * p);
        double er = qtt::plan_seconds(rp);
        // The two models' residuals against 16 measured mid-size cases (d = 14..19,
        // r = 4..48; profiles/r02zzg_fused_decision.json): the fused launch runs
        // ~5 us under its estimate when small and ~30% over it when the estimate
        // passes ~45 us; per-stage plans ran ~1 us per launch over theirs when the
        // stage DP charged 3 us per launch.
        // (The 5 us only up to 4 RHS: at 8-16 RHS the fused launch already runs over
        // its estimate -- d = 13, r = 8 x 16 RHS 37.9 us against 27.5 estimated and 26.7
        // per-stage.)
        ef = ef - (p <= 4 ? 5.0e-6 : 0.0) + 0.6 * std::max(0.0, ef - 27.0e-6);
        er -= 1.0e-6 * double(rp.size());   // the stage DP charges 5 us per launch (it plans better with it); ~4 measured
        if (std::getenv("QTT_DEBUG"))
          std::fprintf(stderr, "qtt: fused plan (%zu stages) at %lld RHS: est %.2f us vs per-stage plan %.2f us\n",
                       fp.size(), (long long)p, ef * 1e6, er * 1e6);
        if (!(ef < er) && !force_fused) break;
        pmax = p;
      }
      if (pmax > 0) {
        h->fstages.resize(fp.size());
        for (size_t s = 0; s < fp.size() && st == QTT_SUCCESS; ++s) {
          h->fstages[s].plan = fp[s];
          st = upload_stage(h, h->fstages[s], cores);
        }
        h->fused_max_nrhs = pmax;
        if (fp.size() > 1) h->max_interior_rank = std::max(h->max_interior_rank, fr);
      }
    }
    if (st == QTT_SUCCESS && shard_bits) {
      qtt::StagePlan& pp = h->proj.plan;
      const int rp = int(h->ranks[dl]), P = 1 << shard_bits;   // padded local top rank
      const int r = int(full_ranks[dl]);
      if (!qtt::projection_plan(rp, shard_bits, h->smem_optin, &pp)) {
        st = QTT_ERROR_NOT_SUPPORTED;
      } else {
        const std::vector<double> Wp = shard_projection(d, full_ranks, full_cores, shard_bits, shard_part);
        h->proj_W = Wp;
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
  } catch (...) {   // no exception may cross the C ABI
    st = QTT_ERROR_CUDA;
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
    const bool capturing = stream_is_capturing(st);
    qtt_status_t so = cached_acquire(&h->ws, &h->ws_bytes, &h->ws_used, h->ws_pending, ws_bytes_for(h, nrhs), st,
                                     capturing, nullptr);
    if (so == QTT_SUCCESS) so = enqueue(h, x_local, send, nrhs, h->ws, st);
    if (so == QTT_SUCCESS) so = cached_release(h->ws_used, &h->ws_pending, st, capturing);
    return so;
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_shard_set_peers(qtt_handle_t h, double* const* recv, int parts) {
  if (!h || !recv || h->shard_bits == 0 || parts != (1 << h->shard_bits)) return QTT_ERROR_INVALID_VALUE;
  for (int g = 0; g < parts; ++g)
    if (!recv[g] || (reinterpret_cast<uintptr_t>(recv[g]) % 16)) return QTT_ERROR_INVALID_VALUE;
  try {
    DeviceGuard gd(h->device);
    if (!h->proj_fused.d_bpack) {   // the projection as a wide stage with the scatter epilogue
      qtt::StagePlan& pp = h->proj_fused.plan;
      const int rp = int(h->ranks[h->d]), r = int(h->proj_W.size() / size_t(parts));
      if (!qtt::projection_plan_wide(rp, h->shard_bits, h->smem_optin, &pp)) return QTT_ERROR_NOT_SUPPORTED;
      const std::vector<double>& Wp = h->proj_W;
      const std::vector<double> pk =
          pack_wide_fn(pp, [&](int kk, int n) { return (kk < r && n < parts) ? Wp[size_t(n) * r + kk] : 0.0; });
      cudaError_t e = qtt::wide_prepare(pp.NB, h->smem_optin);
      if (e == cudaSuccess) e = cudaMalloc(&h->proj_fused.d_bpack, pk.size() * sizeof(double));
      if (e == cudaSuccess)
        e = cudaMemcpy(h->proj_fused.d_bpack, pk.data(), pk.size() * sizeof(double), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {   // leave no half-built projection behind
        if (h->proj_fused.d_bpack) cudaFree(h->proj_fused.d_bpack);
        h->proj_fused.d_bpack = nullptr;
        return from_cuda(e);
      }
      h->proj_fused.ctas_per_sm = 1;
    }
    if (!h->d_peers) {
      cudaError_t e = cudaMalloc(&h->d_peers, size_t(parts) * sizeof(double*));
      if (e != cudaSuccess) return from_cuda(e);
    }
    return from_cuda(cudaMemcpy(h->d_peers, recv, size_t(parts) * sizeof(double*), cudaMemcpyHostToDevice));
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_shard_apply_fused(qtt_handle_t h, const double* x_local, int64_t nrhs, qtt_stream_t stream) {
  if (!h || !x_local || nrhs < 1 || h->shard_bits == 0 || !h->d_peers) return QTT_ERROR_INVALID_VALUE;
  if (nrhs > (int64_t(1) << 31) / (h->N << h->shard_bits)) return QTT_ERROR_NOT_SUPPORTED;
  if ((reinterpret_cast<uintptr_t>(x_local) % 16) || !is_device_ptr(x_local, h->device))
    return QTT_ERROR_NOT_SUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    const bool capturing = stream_is_capturing(st);
    qtt_status_t so = cached_acquire(&h->ws, &h->ws_bytes, &h->ws_used, h->ws_pending, ws_bytes_for(h, nrhs), st,
                                     capturing, nullptr);
    if (so == QTT_SUCCESS) so = enqueue(h, x_local, nullptr, nrhs, h->ws, st, true);
    if (so == QTT_SUCCESS) so = cached_release(h->ws_used, &h->ws_pending, st, capturing);
    return so;
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_shard_reduce(const double* recv, double* y_local, int parts, int64_t count, qtt_stream_t stream) {
  if (!recv || !y_local || parts < 1 || count < 2 || (count % 2)) return QTT_ERROR_INVALID_VALUE;
  if ((reinterpret_cast<uintptr_t>(recv) % 16) || (reinterpret_cast<uintptr_t>(y_local) % 16))
    return QTT_ERROR_NOT_SUPPORTED;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return QTT_ERROR_CUDA;
  return from_cuda(qtt::launch_shard_reduce(recv, y_local, parts, count, reinterpret_cast<cudaStream_t>(stream), sms));
}

qtt_status_t qtt_ipc_alloc(size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return QTT_ERROR_INVALID_VALUE;
  *ptr = nullptr;
  return from_cuda(cudaMalloc(ptr, bytes));
}

qtt_status_t qtt_ipc_free(void* ptr) { return ptr ? from_cuda(cudaFree(ptr)) : QTT_SUCCESS; }

qtt_status_t qtt_ipc_get_handle(void* ptr, unsigned char* handle64) {
  if (!ptr || !handle64) return QTT_ERROR_INVALID_VALUE;
  cudaIpcMemHandle_t hd;
  const cudaError_t e = cudaIpcGetMemHandle(&hd, ptr);
  if (e != cudaSuccess) return from_cuda(e);
  static_assert(sizeof(hd) == 64, "CUDA IPC handles are 64 bytes");
  std::memcpy(handle64, &hd, 64);
  return QTT_SUCCESS;
}

qtt_status_t qtt_ipc_open(const unsigned char* handle64, void** ptr) {
  if (!handle64 || !ptr) return QTT_ERROR_INVALID_VALUE;
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle64, 64);
  *ptr = nullptr;
  return from_cuda(cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess));
}

qtt_status_t qtt_ipc_close(void* ptr) { return ptr ? from_cuda(cudaIpcCloseMemHandle(ptr)) : QTT_SUCCESS; }

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

qtt_status_t qtt_stage_super_core(int d, const int64_t* ranks, const double* const* cores, int k_first,
                                  int k_last, double* W) {
  if (d < 1 || d > 30 || !ranks || !cores || !W || k_first < 1 || k_last > d || k_first > k_last ||
      k_last - k_first + 1 > 12)
    return QTT_ERROR_INVALID_VALUE;
  for (int k = k_first - 1; k <= k_last; ++k)
    if (ranks[k] < 1 || ranks[k] > 4096) return QTT_ERROR_INVALID_VALUE;
  for (int k = k_first - 1; k < k_last; ++k)
    if (!cores[k]) return QTT_ERROR_INVALID_VALUE;
  try {
    const std::vector<double> w = super_core(cores, ranks, k_first, k_last);
    std::copy(w.begin(), w.end(), W);
  } catch (...) {
    return QTT_ERROR_OUT_OF_MEMORY;
  }
  return QTT_SUCCESS;
}

// graphs captured on a released cached workspace are stale
static void drop_graphs_on(qtt_plan* h, const void* old_ws) {
  for (size_t i = h->graphs.size(); i-- > 0;)
    if (h->graphs[i].ws == old_ws) {
      cudaGraphExecDestroy(h->graphs[i].exec);
      h->graphs.erase(h->graphs.begin() + i);
    }
}

qtt_status_t qtt_workspace_size(qtt_handle_t h, int64_t nrhs, size_t* bytes) {
  if (!h || !bytes || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  *bytes = ws_bytes_for(h, h->shard_bits ? nrhs : rhs_group(h, nrhs));
  return QTT_SUCCESS;
}

// Enqueue y = A x for nrhs RHS as consecutive groups of `group` RHS sharing
// one workspace (stream order serialises the groups).  One group replays the
// cached CUDA graph; several use plain launches (a graph per group pointer
// pair would only churn the cache at these sizes).
static qtt_status_t enqueue_groups(qtt_plan* h, const double* x, double* y, int64_t nrhs, int64_t group, void* ws,
                                   cudaStream_t st, bool bar_zero = false) {
  if (group >= nrhs && use_fused(h, nrhs)) {
    // a cooperative launch is cheaper from a cached graph; the default
    // (non-cooperative, PDL) launch runs back to back with the previous kernel
    if (qtt::fused_cooperative()) return enqueue_graphed(h, x, y, nrhs, ws, st, bar_zero ? 1 : 2);
    return enqueue_fused(h, x, y, nrhs, ws, st, !bar_zero);
  }
  if (group >= nrhs) return enqueue_graphed(h, x, y, nrhs, ws, st);
  for (int64_t r0 = 0; r0 < nrhs; r0 += group) {
    const int64_t g = std::min(group, nrhs - r0);
    const size_t off = size_t(r0) * size_t(h->N);
    const qtt_status_t s = enqueue(h, x + off, y + off, g, ws, st);
    if (s != QTT_SUCCESS) return s;
  }
  return QTT_SUCCESS;
}

// RHS per group for an apply on the cached workspace: rhs_group, lowered
// further while the workspace for the group would not fit in the device
// memory free now (plus the cached block it replaces).
static int64_t cached_group(qtt_plan* h, int64_t nrhs) {
  int64_t g = rhs_group(h, nrhs);
  if (ws_bytes_for(h, g) <= h->ws_bytes) return g;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return g;
  }
  const double avail = 0.92 * double(free_b + h->ws_bytes);
  while (g > 1 && double(ws_bytes_for(h, g)) > avail) g = (g + 1) / 2;
  return g;
}

qtt_status_t qtt_apply_ws(qtt_handle_t h, const double* x, double* y, int64_t nrhs, void* ws,
                          size_t ws_bytes, qtt_stream_t stream) {
  qtt_status_t s = check_apply_args(h, x, y, nrhs);
  if (s != QTT_SUCCESS) return s;
  const size_t need = ws_bytes_for(h, rhs_group(h, nrhs));
  if (!ws || ws_bytes < need) return QTT_ERROR_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(ws) % 256) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(ws)) return QTT_ERROR_NOT_SUPPORTED;
  try {
    DeviceGuard g(h->device);
    return enqueue_groups(h, x, y, nrhs, rhs_group(h, nrhs), ws, reinterpret_cast<cudaStream_t>(stream));
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

#ifdef QTT_HOST_PROFILE   // diagnostic build: host time per step of qtt_apply, printed every 2000 calls
struct HostProf {
  double t[8] = {};
  long n = 0;
  std::chrono::steady_clock::time_point last;
  void mark(int i) {
    const auto now = std::chrono::steady_clock::now();
    if (i > 0) t[i] += std::chrono::duration<double, std::micro>(now - last).count();
    last = now;
  }
  void done() {
    if (++n % 500) return;
    std::fprintf(stderr, "qtt host us/call: args %.2f guard+capq %.2f group %.2f acquire %.2f enqueue %.2f release %.2f\n",
                 t[1] / n, t[2] / n, t[3] / n, t[4] / n, t[5] / n, t[6] / n);
  }
};
static HostProf hprof;
#define HP(i) hprof.mark(i)
#else
#define HP(i)
#endif

qtt_status_t qtt_apply(qtt_handle_t h, const double* x, double* y, int64_t nrhs, qtt_stream_t stream) {
  HP(0);
  qtt_status_t s = check_apply_args(h, x, y, nrhs);
  HP(1);
  if (s != QTT_SUCCESS) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    const bool capturing = stream_is_capturing(st);
    HP(2);
    void* old_ws = h->ws;
    bool grew = false;
    int64_t group = cached_group(h, nrhs);
    HP(3);
    qtt_status_t so = cached_acquire(&h->ws, &h->ws_bytes, &h->ws_used, h->ws_pending, ws_bytes_for(h, group), st,
                                     capturing, &grew);
    HP(4);
    while (so == QTT_ERROR_OUT_OF_MEMORY && group > 1 && !capturing) {   // smaller RHS groups
      group = (group + 1) / 2;
      bool g2 = false;
      so = cached_acquire(&h->ws, &h->ws_bytes, &h->ws_used, h->ws_pending, ws_bytes_for(h, group), st, false, &g2);
      grew = grew || g2;
    }
    if (grew) {
      drop_graphs_on(h, old_ws);
      h->ws_header_zero = false;
    }
    // the cached workspace's grid-barrier words stay 0 once cleared (every
    // fused launch leaves them so; per-stage applies clear the whole header)
    if (so == QTT_SUCCESS) so = enqueue_groups(h, x, y, nrhs, group, h->ws, st, h->ws_header_zero);
    HP(5);
    if (so == QTT_SUCCESS) h->ws_header_zero = true;
    if (so == QTT_SUCCESS) so = cached_release(h->ws_used, &h->ws_pending, st, capturing);
    HP(6);
#ifdef QTT_HOST_PROFILE
    hprof.done();
#endif
    return so;
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

}  // extern "C"

namespace qtt {
namespace rt {
qtt_status_t grid_apply_fused(qtt_plan* h, const double* grid_in, double* grid_out, int64_t nrhs, int dim,
                              cudaStream_t st) {
  if (!use_fused(h, nrhs) || rhs_group(h, nrhs) < nrhs) return QTT_ERROR_NOT_SUPPORTED;
  qtt_status_t s = check_apply_args(h, grid_in, grid_out, nrhs);
  if (s != QTT_SUCCESS) return s;
  const bool capturing = stream_is_capturing(st);
  void* old_ws = h->ws;
  bool grew = false;
  s = cached_acquire(&h->ws, &h->ws_bytes, &h->ws_used, h->ws_pending, ws_bytes_for(h, nrhs), st, capturing, &grew);
  if (grew) {
    drop_graphs_on(h, old_ws);
    h->ws_header_zero = false;
  }
  if (s == QTT_SUCCESS) s = enqueue_fused(h, grid_in, grid_out, nrhs, h->ws, st, !h->ws_header_zero, dim);
  if (s == QTT_SUCCESS) h->ws_header_zero = true;
  if (s == QTT_SUCCESS) s = cached_release(h->ws_used, &h->ws_pending, st, capturing);
  return s;
}
}  // namespace rt
}  // namespace qtt

extern "C" {

qtt_status_t qtt_apply_host(qtt_handle_t h, const double* x_host, double* y_host, int64_t nrhs,
                            qtt_stream_t stream) {
  if (!h || !x_host || !y_host || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  try {
    DeviceGuard g(h->device);
    // staging for one group of RHS at a time (bounded by rhs_group and by
    // the device memory the group's workspace needs)
    const int64_t group = std::min(cached_group(h, nrhs), rhs_group(h, nrhs));
    const size_t elems = size_t(h->N) * size_t(group);
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
    // pipelined copies: one RHS, at least two stages, enough rows to chunk --
    // and not a latency-bound size the fused apply runs in one launch (the
    // same plan as qtt_apply, so both give the same bits)
    if (nrhs == 1 && h->stages.size() >= 2 && h->shard_bits == 0 && !h->timing && !use_fused(h, 1) &&
        (h->N >> (h->stages.front().plan.k1 - h->stages.front().plan.k0 + 1)) >= 8 * 64 &&
        (h->N >> (h->stages.back().plan.k1 - h->stages.back().plan.k0 + 1)) >= 8 * 64) {
      void* old_ws = h->ws;
      bool grew = false;
      qtt_status_t s = cached_acquire(&h->ws, &h->ws_bytes, &h->ws_used, h->ws_pending, ws_bytes_for(h, 1), st,
                                      false, &grew);
      if (grew) drop_graphs_on(h, old_ws);
      if (s == QTT_SUCCESS) s = apply_host_pipelined(h, x_host, y_host, st);
      if (s == QTT_SUCCESS) h->ws_header_zero = true;      // the pipelined apply cleared the header
      if (s == QTT_SUCCESS) s = cached_release(h->ws_used, &h->ws_pending, st, false);
      if (s != QTT_SUCCESS) return s;
      return from_cuda(cudaStreamSynchronize(st));
    }
    for (int64_t r0 = 0; r0 < nrhs; r0 += group) {
      const int64_t gr = std::min(group, nrhs - r0);
      const size_t off = size_t(r0) * size_t(h->N), n = size_t(gr) * size_t(h->N);
      cudaError_t e = cudaMemcpyAsync(h->hx, x_host + off, n * sizeof(double), cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return from_cuda(e);
      qtt_status_t s = qtt_apply(h, h->hx, h->hy, gr, stream);
      if (s != QTT_SUCCESS) return s;
      e = cudaMemcpyAsync(y_host + off, h->hy, n * sizeof(double), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return from_cuda(e);
    }
    return from_cuda(cudaStreamSynchronize(st));
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
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

qtt_status_t qtt_get_apply_plan(qtt_handle_t h, int64_t nrhs, int* launches, int* n_stages, int* k_first,
                                int* k_last, int* variant) {
  if (!h || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  const int64_t group = h->shard_bits ? nrhs : rhs_group(h, nrhs);
  const int64_t groups = (nrhs + group - 1) / group;
  const bool fused = group >= nrhs && use_fused(h, nrhs);
  const std::vector<Stage>& S = fused ? h->fstages : h->stages;
  int per = fused ? 1 : 0;
  if (!fused)
    for (const Stage& st : S) per += 1 + (stage_ksplit(h, st, 0) > 1 ? 1 : 0);
  if (h->shard_bits) per += 1;
  if (launches) *launches = int(std::min<int64_t>(int64_t(per) * groups, 0x7fffffff));
  if (n_stages) *n_stages = int(S.size());
  for (size_t i = 0; i < S.size(); ++i) {
    if (k_first) k_first[i] = S[i].plan.k0;
    if (k_last) k_last[i] = S[i].plan.k1;
    if (variant) variant[i] = fused ? int(qtt::kFused) : S[i].plan.variant;
  }
  return QTT_SUCCESS;
}

qtt_status_t qtt_set_fused(qtt_handle_t h, int enable) {
  if (!h) return QTT_ERROR_INVALID_VALUE;
  h->fused_on = enable != 0;
  return QTT_SUCCESS;
}

qtt_status_t qtt_get_stage_split(qtt_handle_t h, int s, int64_t nrhs, int* ksplit) {
  if (!h || !ksplit || nrhs < 1) return QTT_ERROR_INVALID_VALUE;
  if (h->shard_bits && s == int(h->stages.size())) {
    *ksplit = 1;
    return QTT_SUCCESS;
  }
  if (s < 0 || s >= int(h->stages.size())) return QTT_ERROR_INVALID_VALUE;
  const Stage& S = h->stages[s];
  *ksplit = stage_ksplit(h, S, nrhs * (int64_t(1) << (h->d - (S.plan.k1 - S.plan.k0 + 1))));
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
  // every plain enqueue records `last`; the cached buffers' events cover the
  // work around an apply that uses them (grid pack/unpack, host copies)
  if (h->last) cudaEventSynchronize(h->last);
  if (h->ws_pending) cudaEventSynchronize(h->ws_used);
  if (h->g_pending) cudaEventSynchronize(h->g_used);
  free_plan(h);
  return QTT_SUCCESS;
}

}  // extern "C"
