// DMMA vs DFMA issue-capacity probe (VERDICT r1 "settle the DMMA question").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe tools/dmma_probe.cu
//   ./dmma_probe            -> one JSON line per variant
//
// Variants (every CTA 256 threads, grid = 148 * occupancy):
//   dfma      : 8 independent DFMA chains per thread
//   dmma      : 4 independent mma.sync.m8n8k4.f64 accumulators per warp
//   split     : warps 0-3 of each CTA run the DMMA loop, warps 4-7 the DFMA loop
//   interleave: every warp alternates one DMMA with 8 DFMAs
// If DMMA and DFMA share one datapath, split/interleave reach the single-
// pipe rate; if DMMA has its own issue capacity they add up.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(256) k_probe(long long iters, double seed, double* out) {
  const int warp = threadIdx.x >> 5;
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed + 1e-3 * (threadIdx.x + i);
  double acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = seed * i;
  const double a = 1.0 - 1e-9 * threadIdx.x, b = 1e-7 * (threadIdx.x & 7);
  const bool do_mma = MODE == 1 || (MODE == 2 && warp < 4) || MODE == 3;
  const bool do_fma = MODE == 0 || (MODE == 2 && warp >= 4) || MODE == 3;
  for (long long it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(acc[i], a, b);
    }
    if (do_fma) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"dfma", "dmma", "split", "interleave"};
  void (*ks[4])(long long, double, double*) = {k_probe<0>, k_probe<1>, k_probe<2>, k_probe<3>};
  for (int occ = 1; occ <= 4; occ *= 2) {
    const int grid = nsm * occ;
    for (int m = 0; m < 4; ++m) {
      const long long iters = 20000;
      ks[m]<<<grid, 256>>>(100, 1.0, out);
      cudaEventRecord(e0);
      ks[m]<<<grid, 256>>>(iters, 1.0, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = grid * 8.0;
      // per warp-iteration: DMMA 4 x 512 flop (m8n8k4: 2*8*8*4), DFMA 32 x 32 lanes x 2 flop
      double mma_flop = 0, fma_flop = 0;
      const double wm = (m == 1 || m == 3) ? warps : (m == 2 ? warps / 2 : 0);
      const double wf = (m == 0 || m == 3) ? warps : (m == 2 ? warps / 2 : 0);
      mma_flop = wm * iters * 4 * 512.0;
      fma_flop = wf * iters * 32 * 32 * 2.0;
      const double s = ms * 1e-3;
      printf("{\"variant\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, "
             "\"total_tflops\": %.2f, \"sm_clock_mhz_attr\": %d}\n",
             names[m], occ, ms, mma_flop / s * 1e-12, fma_flop / s * 1e-12, (mma_flop + fma_flop) / s * 1e-12,
             clk / 1000);
    }
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
