// C ABI of libqtt_b200.so, the NEXT rows (include/qtt.h): Morton ordering and
// the grid apply (NEXT-2), the QTT-compressed matvec (NEXT-3), products of
// operators (NEXT-1).
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

using namespace qtt::rt;

extern "C" {

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
    // a fused apply gathers / scatters the Morton order in its first / last
    // stage: one launch, no staging vectors
    if (use_fused(h, nrhs) && rhs_group(h, nrhs) >= nrhs) {
      const qtt_status_t fs = grid_apply_fused(h, grid_in, grid_out, nrhs, dim, st);
      // a refused cooperative launch disables the fused plan: take the staged path below
      if (fs != QTT_ERROR_NOT_SUPPORTED || use_fused(h, nrhs)) return fs;
    }
    const size_t elems = size_t(h->N) * size_t(nrhs);
    const bool capturing = stream_is_capturing(st);
    // the staging vectors are shared by the handle's grid applies: order this
    // one after the previous (on any stream) before the pack overwrites gx
    void* gbuf = h->gx;
    size_t gbytes = h->g_elems * 2 * sizeof(double);
    qtt_status_t s = cached_acquire(&gbuf, &gbytes, &h->g_used, h->g_pending, elems * 2 * sizeof(double), st,
                                    capturing, nullptr);
    if (s != QTT_SUCCESS) return s;
    h->g_elems = gbytes / (2 * sizeof(double));
    h->gx = static_cast<double*>(gbuf);
    h->gy = h->gx + h->g_elems;
    s = qtt_morton_pack(grid_in, h->gx, dim, levels, nrhs, stream);
    if (s == QTT_SUCCESS) s = qtt_apply(h, h->gx, h->gy, nrhs, stream);
    if (s == QTT_SUCCESS) s = qtt_morton_unpack(h->gy, grid_out, dim, levels, nrhs, stream);
    if (s == QTT_SUCCESS) s = cached_release(h->g_used, &h->g_pending, st, capturing);
    return s;
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
    // one grow-only scratch per handle: b's cores | product cores (unless the
    // caller's) | densify workspace.  Allocating per call (stream-ordered
    // allocator, release threshold 0) re-mapped ~45 MB each time: 13 ms.
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t vb = al(std::max<size_t>(boff[d], 1) * sizeof(double));
    const size_t cb = c_cores ? 0 : al(coff[d] * sizeof(double));
    const size_t wsb = c_dense ? qtt::densify_workspace_bytes(d, R.data()) : 0;
    cudaError_t e = cudaSuccess;
    if (vb + cb + wsb > h->cmv_bytes) {
      // the scratch is only touched by this synchronous call: no pending work uses it
      if (h->cmv) cudaFree(h->cmv);
      h->cmv = nullptr;
      h->cmv_bytes = 0;
      e = cudaMalloc(&h->cmv, vb + cb + wsb);
      if (e != cudaSuccess) {
        h->cmv = nullptr;
        return from_cuda(e);
      }
      h->cmv_bytes = vb + cb + wsb;
    }
    unsigned char* base = static_cast<unsigned char*>(h->cmv);
    double* dV = reinterpret_cast<double*>(base);
    double* dC = c_cores ? c_cores : reinterpret_cast<double*>(base + vb);
    void* ws = wsb ? base + vb + cb : nullptr;
    // b's cores: host -> device in one copy (pageable; the host arrays may be freed on return)
    std::vector<double> hv(std::max<size_t>(boff[d], 1));
    for (int k = 0; k < d; ++k)
      std::copy(b_cores[k], b_cores[k] + (boff[k + 1] - boff[k]), hv.begin() + boff[k]);
    e = cudaMemcpyAsync(dV, hv.data(), boff[d] * sizeof(double), cudaMemcpyHostToDevice, st);
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
  *bytes = product_ws_bytes(p, rhs_group(p->factors[0], nrhs));
  return QTT_SUCCESS;
}

qtt_status_t qtt_product_apply_ws(qtt_product_t p, const double* x, double* y, int64_t nrhs, void* ws,
                                  size_t ws_bytes, qtt_stream_t stream) {
  if (!p) return QTT_ERROR_INVALID_VALUE;
  qtt_status_t s = check_apply_args(p->factors[0], x, y, nrhs);
  if (s != QTT_SUCCESS) return s;
  // RHS in groups of rhs_group (N * group <= 2^31 rows per launch)
  const int64_t group = rhs_group(p->factors[0], nrhs);
  const size_t need = product_ws_bytes(p, group);
  if (!ws || ws_bytes < need) return QTT_ERROR_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(ws) % 256) return QTT_ERROR_NOT_SUPPORTED;
  if (!is_device_ptr(ws)) return QTT_ERROR_NOT_SUPPORTED;
  try {
    DeviceGuard g(p->device);
    const int n = int(p->factors.size());
    unsigned char* base = static_cast<unsigned char*>(ws);
    const size_t vb = product_vec_bytes(p, group);
    double* tmp[2] = {reinterpret_cast<double*>(base), reinterpret_cast<double*>(base + vb)};
    const size_t nvec = n >= 3 ? 2 : (n == 2 ? 1 : 0);
    void* fws = base + nvec * vb;
    for (int64_t r0 = 0; r0 < nrhs; r0 += group) {
      const int64_t gr = std::min(group, nrhs - r0);
      const size_t off = size_t(r0) * size_t(p->N);
      const double* in = x + off;
      // F_{n-1} first; each factor's stages read the previous factor's output
      for (int i = n - 1, step = 0; i >= 0; --i, ++step) {
        double* out = (i == 0) ? y + off : tmp[step & 1];
        // each factor runs the plan a plain apply of it would (fused one-launch or per-stage)
        s = use_fused(p->factors[i], gr)
                ? enqueue_fused(p->factors[i], in, out, gr, fws, reinterpret_cast<cudaStream_t>(stream), true)
                : enqueue(p->factors[i], in, out, gr, fws, reinterpret_cast<cudaStream_t>(stream));
        if (s != QTT_SUCCESS) return s;
        in = out;
      }
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
    const bool capturing = stream_is_capturing(st);
    qtt_status_t s2 = cached_acquire(&p->ws, &p->ws_bytes, &p->ws_used, p->ws_pending,
                                     product_ws_bytes(p, rhs_group(p->factors[0], nrhs)),
                                     st, capturing, nullptr);
    if (s2 == QTT_SUCCESS) s2 = qtt_product_apply_ws(p, x, y, nrhs, p->ws, p->ws_bytes, stream);
    if (s2 == QTT_SUCCESS) s2 = cached_release(p->ws_used, &p->ws_pending, st, capturing);
    return s2;
  } catch (...) {
    return QTT_ERROR_CUDA;
  }
}

qtt_status_t qtt_product_destroy(qtt_product_t p) {
  if (!p) return QTT_SUCCESS;
  DeviceGuard g(p->device);
  if (p->ws_pending) cudaEventSynchronize(p->ws_used);
  if (p->ws) cudaFree(p->ws);
  if (p->ws_used) cudaEventDestroy(p->ws_used);
  delete p;
  return QTT_SUCCESS;
}

}  // extern "C"
