// FP64 peak probe for B200 (sm_100a): SURVEY.md §7 step 0 ("B0 peaks probe").
//
// MEASURED_PEAKS.json carries HBM copy bandwidth and bf16 GEMM throughput but
// no FP64 figure, and the QTT apply (Alg. 2) is an FP64
// contraction.  This standalone program measures, with CUDA events:
//   * DFMA  : CUDA-core fp64 FMA burn (independent chains, full grid)
//   * DMMA  : mma.sync f64 burn for m8n8k4, m16n8k4, m16n8k8, m16n8k16
//   * copy  : fp64 device-to-device streaming copy (read+write bytes)
// and prints one JSON object.  It is a measurement tool, not part of the
// product path.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void dfma_burn(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
__device__ __forceinline__ void mma_step(double (&d)[4], const double (&a)[8], const double (&b)[4]);

// SHAPE 0: m8n8k4 (uses d[0..1], a[0], b[0])
template <> __device__ __forceinline__ void mma_step<0>(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a[0]), "d"(b[0]));
}
// SHAPE 1: m16n8k4
template <> __device__ __forceinline__ void mma_step<1>(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
// SHAPE 2: m16n8k8
template <> __device__ __forceinline__ void mma_step<2>(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
// SHAPE 3: m16n8k16
template <> __device__ __forceinline__ void mma_step<3>(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE, int NACC>
__global__ void dmma_burn(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  double d[NACC][4];
#pragma unroll
  for (int c = 0; c < NACC; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NACC; ++c) mma_step<SHAPE>(d[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NACC; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// Mixed probe: even warps issue DMMA m8n8k4 chains, odd warps DFMA chains, in
// the same CTAs.  If DMMA and DFMA run on separate units the combined rate
// exceeds either alone; if they share the FP64 pipe it does not.
__global__ void mixed_burn(double* out, int dmma_iters, int dfma_iters, double fa, double fb) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if ((warp & 1) == 0) {
    double a = 1e-3 * threadIdx.x, b = 1e-3 * (threadIdx.x + 1);
    double d[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = 0.0;
    for (int it = 0; it < dmma_iters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  } else {
    double acc[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-9 + c;
    for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], fa, fb);
      }
    }
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c];
  }
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_f64(const double2* __restrict__ in, double2* __restrict__ out, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n2; i += stride) out[i] = in[i];
}

template <typename F>
static float time_ms(F launch, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, (size_t)sms * 64 * 1024 * sizeof(double)));
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz\": %d,\n",
         p.name, sms, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate);

  // DFMA: blocks = sms*8, 256 threads, kChains*8 fma per iter per thread
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    float ms = time_ms([&] { dfma_burn<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double flops = 2.0 * (double)blocks * threads * iters * 8 * kChains;
    printf(" \"dfma_tflops\": %.3f,\n", flops / ms * 1e-9);
  }
  // DMMA shapes
  const int mnk[4][3] = {{8, 8, 4}, {16, 8, 4}, {16, 8, 8}, {16, 8, 16}};
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  for (int s = 0; s < 4; ++s) {
    for (int wpb : {4, 8, 16}) {
      int iters = 2048 >> (s == 3 ? 2 : (s == 2 ? 1 : 0));
      int blocks = sms * 4, threads = 32 * wpb;
      constexpr int NA = 8;
      float ms;
      auto L = [&] {
        switch (s) {
          case 0: dmma_burn<0, NA><<<blocks, threads>>>(out, iters); break;
          case 1: dmma_burn<1, NA><<<blocks, threads>>>(out, iters); break;
          case 2: dmma_burn<2, NA><<<blocks, threads>>>(out, iters); break;
          default: dmma_burn<3, NA><<<blocks, threads>>>(out, iters); break;
        }
      };
      ms = time_ms(L, 5);
      double flops = 2.0 * mnk[s][0] * mnk[s][1] * mnk[s][2] * (double)NA * iters * (double)blocks * wpb;
      printf(" \"dmma_%s_w%d_tflops\": %.3f,\n", names[s], wpb, flops / ms * 1e-9);
    }
  }
  // mixed DMMA + DFMA (separate units or one FP64 pipe?)
  for (int ratio : {1, 2, 4}) {
    // per warp: DMMA warp does 8*dmma_iters m8n8k4 (512 flop each); DFMA warp does
    // 64*dfma_iters fma per thread (64 flop per warp-instr pair... 2*32 per instr)
    int blocks = sms * 4, threads = 32 * 16;
    int dmma_iters = 2048, dfma_iters = 2048 * 8 * 512 / (64 * 2 * 32) / ratio;
    float ms = time_ms([&] { mixed_burn<<<blocks, threads>>>(out, dmma_iters, dfma_iters, 0.999999, 1e-7); }, 5);
    double warps = (double)blocks * 16 / 2;
    double f_dmma = warps * dmma_iters * 8 * 512.0;
    double f_dfma = warps * 32.0 * dfma_iters * 8 * kChains * 2.0;
    printf(" \"mixed_r%d_total_tflops\": %.3f, \"mixed_r%d_dmma_share\": %.3f,\n", ratio,
           (f_dmma + f_dfma) / ms * 1e-9, ratio, f_dmma / (f_dmma + f_dfma));
  }
  // copy
  {
    size_t bytes = (size_t)4 << 30;  // 4 GiB each
    double2 *a, *b;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes));
    size_t n2 = bytes / sizeof(double2);
    float ms = time_ms([&] { copy_f64<<<sms * 8, 512>>>(a, b, n2); }, 10);
    printf(" \"copy_kernel_gbs\": %.1f,\n", 2.0 * bytes / ms * 1e-6);
    float ms2 = time_ms([&] { CK(cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice)); }, 10);
    printf(" \"copy_memcpy_gbs\": %.1f\n", 2.0 * bytes / ms2 * 1e-6);
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  printf("}\n");
  return 0;
}
