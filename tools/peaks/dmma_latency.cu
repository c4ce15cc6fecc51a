// DMMA.8x8x4 latency / per-sub-partition throughput probe (sm_100a).
// One CTA per SM with W warps (W = 1: one sub-partition; W = 4: one warp per
// sub-partition), each warp running NA independent accumulator chains of
// mma.sync.m8n8k4.f64.  clock64 cycles per DMMA per warp: NA = 1 gives the
// dependent-issue latency, large NA the throughput.  Also the L2-hit latency
// of dependent ld.global.cg loads (pointer chase).  Measurement tool only.
#include <cstdio>
#include <cuda_runtime.h>

template <int NA>
__global__ void chain(double* out, long long* cyc, int iters) {
  double a = 1e-3 * threadIdx.x, b = 2e-3;
  double d[NA][2];
#pragma unroll
  for (int c = 0; c < NA; ++c) d[c][0] = d[c][1] = 0.0;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NA; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < NA; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

__global__ void chase(const unsigned* next, long long* cyc, int iters, unsigned* sink) {
  unsigned p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  sink[0] = p;
  cyc[0] = t1 - t0;
}

template <int NA>
void run(int warps, double* out, long long* cyc) {
  const int iters = 4096;
  chain<NA><<<148, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, sizeof(long long) * warps, cudaMemcpyDeviceToHost);
  printf("  \"w%d_na%d_cycles_per_dmma\": %.2f,\n", warps, NA, double(h[0]) / (double(iters) * NA));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMalloc(&cyc, 64 * sizeof(long long));
  printf("{\n");
  for (int w : {1, 4, 8}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
    run<16>(w, out, cyc);
  }
  // L2-hit pointer chase: 16 MB ring (fits L2), stride 4 KB + 1 line
  const int n = 4 << 20;
  unsigned* h = new unsigned[n];
  for (int i = 0; i < n; ++i) h[i] = unsigned((i + 1056) % n);
  unsigned *dn, *sink;
  cudaMalloc(&dn, n * sizeof(unsigned));
  cudaMalloc(&sink, 16);
  cudaMemcpy(dn, h, n * sizeof(unsigned), cudaMemcpyHostToDevice);
  chase<<<1, 1>>>(dn, cyc, 1000, sink);   // warm
  chase<<<1, 1>>>(dn, cyc, 4000, sink);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("  \"l2_hit_chase_cycles\": %.1f\n}\n", double(c) / 4000);
  return 0;
}
