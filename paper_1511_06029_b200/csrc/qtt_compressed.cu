// QTT-compressed matrix-vector product and TT-vector densification (NEXT-3).
//
// PAPER.md section 4.2 "QTT compressed matrix-vector product":
// with b in QTT form (cores G^b_k(beta_{k-1}, j_k, beta_k)), the cores of c = A b are
//   G^c_k(overline{alpha_{k-1} beta_{k-1}}, i_k, overline{alpha_k beta_k})
//       = sum_{j_k} G^A_k(alpha_{k-1}, overline{i_k j_k}, alpha_k) G^b_k(beta_{k-1}, j_k, beta_k)
// (ranks R_k = r^A_k r^b_k, cost O(r_A^2 r_b^2 log N)).  `compressed_cores_kernel`
// computes them, one thread per output entry.
//
// Densification of a TT vector v (Eq. TTdeccores P:519-523 for a vector:
// v[i] = H_1(:, i_1, :) ... H_d(:, i_d, :)), split at level a:
//   L_a[i_1..i_a][beta]       = H_1 ... H_a             (bottom-up, 2^a x R_a)
//   Rt_{a+1}[i_{a+1}..i_d][beta] = (H_{a+1} ... H_d)^T    (top-down, 2^(d-a) x R_a)
//   v[i_low + 2^a i_high]     = sum_beta L_a[i_low][beta] Rt_{a+1}[i_high][beta]
// Every step is a GEMM run by the wide DMMA stage kernel (qtt_wide_kernel.cu)
// with its row-separation epilogue doing the digit bookkeeping:
//   bottom-up step k : A = L_{k-1} (2^(k-1) rows), W[beta][ii*r + b] = H_k[beta][ii][b],
//                      out row m + 2^(k-1) ii      (log2_q = k-1: i_k most significant)
//   top-down step k  : A = Rt_{k+1} (2^(d-k) rows), W[beta][ii*r + b] = H_k[b][ii][beta],
//                      out row 2 m + ii            (log2_q = 0: i_k least significant)
//   final            : A = Rt_{a+1}, W[beta][i_low] = L_a[i_low][beta],
//                      out row 2^a m + i_low       (n_i = 2^a, r_out = 1, log2_q = 0)
// so the dense result costs ~2 R_a N flops plus O(2^(d/2) R^2) for the halves.
// Ranks are padded to multiples of kWideBK (zero rows / columns of W).
#include "qtt_internal.h"

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

namespace qtt {
namespace {

constexpr int kThreads = 256;

// C[(a*rb + beta)][i][(a2*rb2 + beta2)] = sum_j G[a][i][j][a2] V[beta][j][beta2]
__global__ void compressed_cores_kernel(const double* __restrict__ G, const double* __restrict__ V, double* __restrict__ C,
                                        int ra, int ra2, int rb, int rb2) {
  const int64_t R2 = int64_t(ra2) * rb2;
  const int64_t total = int64_t(ra) * rb * 2 * R2;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = t / (2 * R2);
    const int rem = int(t - row * 2 * R2);
    const int i = rem / int(R2);
    const int col = rem - i * int(R2);
    const int a = int(row / rb), beta = int(row - int64_t(a) * rb);
    const int a2 = col / rb2, beta2 = col - a2 * rb2;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 2; ++j)
      acc = fma(G[((int64_t(a) * 2 + i) * 2 + j) * ra2 + a2], V[(int64_t(beta) * 2 + j) * rb2 + beta2], acc);
    C[t] = acc;
  }
}

enum PackMode : int { kBottomUp = 0, kTopDown = 1, kFinal = 2 };

// Wide-kernel B layout (qtt_api.cpp pack_wide):
//   pack[cb][ch][kb][nb][lane][v] = Bmat[ch*32 + kb*16 + 4*(lane%4) + v][(cb*NB + nb)*8 + lane/4]
struct PackArgs {
  int mode;
  const double* src;   // H_k [R_in][2][R_out] (bottom-up / top-down) or L_a [2^a][ld] (final)
  int R_in, R_out;     // real ranks of H_k (bottom-up / top-down); final: R_in = R_a, R_out unused
  int ld;              // final: row length of L_a
  int K, nout, r_out;  // GEMM shape (K padded), columns n = ii * r_out + b
  int NB, nchunks, ncb;
  double* dst;
};

__global__ void pack_kernel(const PackArgs p) {
  const int64_t chunk = int64_t(kWideKBC) * p.NB * 32 * 4;
  const int64_t total = int64_t(p.ncb) * p.nchunks * chunk;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cc = t / chunk;
    int rem = int(t - cc * chunk);
    const int cb = int(cc / p.nchunks), ch = int(cc - int64_t(cb) * p.nchunks);
    const int v = rem & 3;
    rem >>= 2;
    const int lane = rem & 31;
    rem >>= 5;
    const int nb = rem % p.NB, kb = rem / p.NB;
    const int kk = ch * kWideBK + kb * 16 + 4 * (lane & 3) + v;
    const int n = (cb * p.NB + nb) * 8 + (lane >> 2);
    double val = 0.0;
    if (kk < p.K && n < p.nout) {
      if (p.mode == kFinal) {
        if (kk < p.R_in) val = p.src[int64_t(n) * p.ld + kk];
      } else {
        const int ii = n / p.r_out, b = n - ii * p.r_out;
        if (p.mode == kBottomUp) {
          if (kk < p.R_in && b < p.R_out) val = p.src[(int64_t(kk) * 2 + ii) * p.R_out + b];
        } else {  // top-down: Bmat[beta][ii*r + b] = H[b][ii][beta], beta < R_out, b < R_in
          if (kk < p.R_out && b < p.R_in) val = p.src[(int64_t(b) * 2 + ii) * p.R_out + kk];
        }
      }
    }
    p.dst[t] = val;
  }
}

// L_1[i][beta] = H_1[0][i][beta] (bottom) or Rt_d[i][beta] = H_d[beta][i][0] (top), padded rows of ld.
__global__ void seed_kernel(const double* __restrict__ H, double* __restrict__ out, int R, int ld, bool top) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 2 * ld; t += gridDim.x * blockDim.x) {
    const int i = t / ld, beta = t - i * ld;
    double v = 0.0;
    if (beta < R) v = top ? H[(int64_t(beta) * 2 + i) * 1 + 0] : H[int64_t(i) * R + beta];
    out[t] = v;
  }
}

// d = 1: v[i] = H_1[0][i][0]
__global__ void copy2_kernel(const double* __restrict__ H, double* __restrict__ out) {
  if (threadIdx.x < 2) out[threadIdx.x] = H[threadIdx.x];
}

int grid_for(int64_t n, int num_sms) {
  int64_t b = (n + kThreads - 1) / kThreads;
  b = std::min<int64_t>(b, int64_t(num_sms) * 16);
  return int(std::max<int64_t>(b, 1));
}

int pad32(int64_t r) { return int((r + kWideBK - 1) / kWideBK * kWideBK); }

struct WideShape {
  int K, nout, NB, ncb, nchunks;
  size_t pack_elems;
};

WideShape wide_shape(int K, int nout) {
  WideShape w;
  w.K = K;
  w.nout = nout;
  w.NB = nout <= 32 ? 4 : nout <= 64 ? 8 : nout <= 96 ? 12 : 16;
  w.ncb = (nout + 8 * w.NB - 1) / (8 * w.NB);
  w.nchunks = K / kWideBK;
  w.pack_elems = size_t(w.ncb) * w.nchunks * kWideKBC * w.NB * 32 * 4;
  return w;
}

}  // namespace

cudaError_t compressed_cores(int d, const int64_t* ra, const double* const* dG, const int64_t* rb,
                             const double* const* dV, double* const* dC, cudaStream_t st, int num_sms) {
  for (int k = 0; k < d; ++k) {
    const int64_t total = ra[k] * rb[k] * 2 * ra[k + 1] * rb[k + 1];
    compressed_cores_kernel<<<grid_for(total, num_sms), kThreads, 0, st>>>(dG[k], dV[k], dC[k], int(ra[k]),
                                                                           int(ra[k + 1]), int(rb[k]), int(rb[k + 1]));
  }
  return cudaGetLastError();
}

// Workspace bytes tt_densify needs for ranks R[0..d].
size_t densify_workspace_bytes(int d, const int64_t* R) {
  if (d <= 1) return 0;
  const int a = d / 2;
  int rmax = 0;
  for (int k = 1; k < d; ++k) rmax = std::max(rmax, pad32(R[k]));
  const size_t lrows = size_t(1) << a, rrows = size_t(1) << (d - a);
  size_t pack = 0;
  for (int k = 2; k <= a; ++k) pack = std::max(pack, wide_shape(pad32(R[k - 1]), 2 * pad32(R[k])).pack_elems);
  for (int k = d - 1; k >= a + 1; --k) pack = std::max(pack, wide_shape(pad32(R[k]), 2 * pad32(R[k - 1])).pack_elems);
  pack = std::max(pack, wide_shape(pad32(R[a]), 1 << a).pack_elems);
  auto al = [](size_t e) { return (e * sizeof(double) + 255) / 256 * 256; };
  return 256 + 2 * al(lrows * rmax) + 2 * al(rrows * rmax) + al(pack);
}

// v = densify(H_1..H_d) (device cores dH[k] of shape [R_k][2][R_{k+1}]) into out (N doubles).
cudaError_t tt_densify(int d, const int64_t* R, const double* const* dH, double* out, void* ws, cudaStream_t st,
                       int num_sms, size_t smem_optin) {
  if (d == 1) {
    copy2_kernel<<<1, 32, 0, st>>>(dH[0], out);
    return cudaGetLastError();
  }
  const int a = d / 2;
  int rmax = 0;
  for (int k = 1; k < d; ++k) rmax = std::max(rmax, pad32(R[k]));
  const size_t lrows = size_t(1) << a, rrows = size_t(1) << (d - a);
  auto al = [](size_t e) { return (e * sizeof(double) + 255) / 256 * 256; };
  unsigned char* p = static_cast<unsigned char*>(ws);
  int* counters = reinterpret_cast<int*>(p);
  p += 256;
  double* Lb[2] = {reinterpret_cast<double*>(p), reinterpret_cast<double*>(p + al(lrows * rmax))};
  p += 2 * al(lrows * rmax);
  double* Rb[2] = {reinterpret_cast<double*>(p), reinterpret_cast<double*>(p + al(rrows * rmax))};
  p += 2 * al(rrows * rmax);
  double* packed = reinterpret_cast<double*>(p);
  cudaError_t e = cudaMemsetAsync(counters, 0, 256, st);
  if (e != cudaSuccess) return e;
  int ctr = 0;

  auto run = [&](const double* A, double* C, int64_t M, int log2_q, int n_i, int r_out, const WideShape& w) {
    LevelArgs g;
    g.in = A;
    g.out = C;
    g.bpack = packed;
    g.M = M;
    g.log2_q = log2_q;
    g.q = int64_t(1) << log2_q;
    g.n_i = n_i;
    g.tile_counter = counters + (ctr++);
    g.r_out = r_out;
    g.K = w.K;
    g.NB = w.NB;
    g.KB = kWideKBC;
    g.nchunks = w.nchunks;
    g.ncb = w.ncb;
    g.nout = w.nout;
    g.smem = wide_smem_bytes(w.NB);
    const int64_t tiles = (M + kDmmaRowsPerSubtile - 1) / kDmmaRowsPerSubtile * w.ncb;
    g.grid = int(std::min<int64_t>(tiles, num_sms));
    cudaError_t err = wide_prepare(w.NB, smem_optin);
    if (err != cudaSuccess) return err;
    return launch_wide(g, st);
  };
  auto pack = [&](int mode, const double* src, int Rin, int Rout, int ld, const WideShape& w, int r_out) {
    PackArgs pa;
    pa.mode = mode;
    pa.src = src;
    pa.R_in = Rin;
    pa.R_out = Rout;
    pa.ld = ld;
    pa.K = w.K;
    pa.nout = w.nout;
    pa.r_out = r_out;
    pa.NB = w.NB;
    pa.nchunks = w.nchunks;
    pa.ncb = w.ncb;
    pa.dst = packed;
    pack_kernel<<<grid_for(int64_t(w.pack_elems), num_sms), kThreads, 0, st>>>(pa);
    return cudaGetLastError();
  };

  // bottom-up: L_1 .. L_a
  seed_kernel<<<grid_for(2 * pad32(R[1]), num_sms), kThreads, 0, st>>>(dH[0], Lb[0], int(R[1]), pad32(R[1]), false);
  int lcur = 0;
  for (int k = 2; k <= a; ++k) {
    const int Kp = pad32(R[k - 1]), rp = pad32(R[k]);
    const WideShape w = wide_shape(Kp, 2 * rp);
    if ((e = pack(kBottomUp, dH[k - 1], int(R[k - 1]), int(R[k]), 0, w, rp)) != cudaSuccess) return e;
    if ((e = run(Lb[lcur], Lb[lcur ^ 1], int64_t(1) << (k - 1), k - 1, 2, rp, w)) != cudaSuccess) return e;
    lcur ^= 1;
  }
  // top-down: Rt_d .. Rt_{a+1}
  seed_kernel<<<grid_for(2 * pad32(R[d - 1]), num_sms), kThreads, 0, st>>>(dH[d - 1], Rb[0], int(R[d - 1]),
                                                                          pad32(R[d - 1]), true);
  int rcur = 0;
  for (int k = d - 1; k >= a + 1; --k) {
    const int Kp = pad32(R[k]), rp = pad32(R[k - 1]);
    const WideShape w = wide_shape(Kp, 2 * rp);
    if ((e = pack(kTopDown, dH[k - 1], int(R[k - 1]), int(R[k]), 0, w, rp)) != cudaSuccess) return e;
    if ((e = run(Rb[rcur], Rb[rcur ^ 1], int64_t(1) << (d - k), 0, 2, rp, w)) != cudaSuccess) return e;
    rcur ^= 1;
  }
  // final: v[i_low + 2^a i_high] = sum_beta L_a[i_low][beta] Rt_{a+1}[i_high][beta]
  const int Kp = pad32(R[a]);
  const WideShape w = wide_shape(Kp, 1 << a);
  if ((e = pack(kFinal, Lb[lcur], int(R[a]), 0, Kp, w, 1)) != cudaSuccess) return e;
  return run(Rb[rcur], out, int64_t(1) << (d - a), 0, 1 << a, 1, w);
}

}  // namespace qtt
