// Microbenchmark: the eval+solve inner-loop instruction mix (Horner DFMA chain -> DMMA, plus
// DFMA leftover columns) with operands in registers, to separate pipe limits from memory/sync.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// U independent (lambda, m-tile) units per k-step; P planes (Horner depth P-1); REM leftover DFMA
template <int U, int P, int REM>
__global__ void __launch_bounds__(512, 1) mix_kernel(double* out, int iters, double t0) {
  double acc[U][2], accx[U][REM > 0 ? REM : 1];
  double th[P], tl[U], b = 1.0 - threadIdx.x * 1e-5, rv[REM > 0 ? REM : 1];
#pragma unroll
  for (int p = 0; p < P; ++p) th[p] = threadIdx.x * 1e-3 + p;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    acc[u][0] = acc[u][1] = 0.0;
    tl[u] = t0 + u * 1e-3;
#pragma unroll
    for (int c = 0; c < (REM > 0 ? REM : 1); ++c) accx[u][c] = 0.0;
  }
#pragma unroll
  for (int c = 0; c < (REM > 0 ? REM : 1); ++c) rv[c] = 0.5 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double av = th[P - 1];
#pragma unroll
      for (int p = P - 2; p >= 0; --p) av = fma(av, tl[u], th[p]);
      dmma884(acc[u][0], acc[u][1], av, b);
#pragma unroll
      for (int c = 0; c < REM; ++c) accx[u][c] = fma(av, rv[c], accx[u][c]);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) th[p] += 1e-9;  // keep the loads "new" each iteration
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    s += acc[u][0] + acc[u][1];
#pragma unroll
    for (int c = 0; c < REM; ++c) s += accx[u][c];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int U, int P, int REM>
void run(int sms, double* out, int threads) {
  int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dim3 grid(sms);
  mix_kernel<U, P, REM><<<grid, threads>>>(out, iters, 0.3);
  cudaEventRecord(e0);
  mix_kernel<U, P, REM><<<grid, threads>>>(out, iters, 0.3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)grid.x * threads / 32;
  double dmma = 512.0 * U * iters * warps, dfma = 64.0 * U * (P - 1 + REM) * iters * warps;
  // pipe model: DMMA at 37.0, DFMA at 33.6 TF/s sharing one datapath
  double ideal_ms = (dmma / 37.0e12 + dfma / 33.6e12) * 1e3;
  printf("U=%d P=%d REM=%d threads=%d: %.3f ms, pipe-model %.3f ms -> %.1f%%\n", U, P, REM, threads, ms, ideal_ms,
         100.0 * ideal_ms / ms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  run<6, 3, 2>(sms, out, 512);
  run<6, 3, 2>(sms, out, 256);
  run<6, 3, 0>(sms, out, 512);
  run<6, 1, 0>(sms, out, 512);
  run<12, 3, 2>(sms, out, 256);
  run<6, 4, 2>(sms, out, 512);
  run<6, 3, 6>(sms, out, 512);
  return 0;
}
