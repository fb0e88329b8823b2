// Microbenchmark (experiments only): how the FP64 pipe handles the eval+solve instruction mix
// (Horner DFMA -> DMMA + leftover DFMA) depending on instruction order and MMA shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix2 tools/mix2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma16816(double* c, const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__device__ __forceinline__ double vfma(double a, double b, double c) {
  double d;
  asm volatile("fma.rn.f64 %0, %1, %2, %3;\n" : "=d"(d) : "d"(a), "d"(b), "d"(c));
  return d;
}

// MODE 0: compiler order; MODE 1: per unit Horner -> DMMA -> leftover, pinned (volatile);
// MODE 2: all Horners, then all DMMAs, then all leftovers, pinned.
template <int U, int P, int REM, int MODE>
__global__ void __launch_bounds__(512, 1) mix884(double* out, int iters, double t0) {
  double acc[U][2], accx[U][REM > 0 ? REM : 1], av[U];
  double th[P], tl[U], b = 1.0 - threadIdx.x * 1e-5, rv[REM > 0 ? REM : 1];
#pragma unroll
  for (int u = 0; u < U; ++u) av[u] = 0.5 + u;
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
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double a = th[P - 1];
#pragma unroll
        for (int p = P - 2; p >= 0; --p) a = fma(a, tl[u], th[p]);
        dmma884(acc[u][0], acc[u][1], a, b);
#pragma unroll
        for (int c = 0; c < REM; ++c) accx[u][c] = fma(a, rv[c], accx[u][c]);
      }
    } else if (MODE == 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double a = th[P - 1];
#pragma unroll
        for (int p = P - 2; p >= 0; --p) a = vfma(a, tl[u], th[p]);
        dmma884(acc[u][0], acc[u][1], a, b);
#pragma unroll
        for (int c = 0; c < REM; ++c) accx[u][c] = vfma(a, rv[c], accx[u][c]);
      }
    } else if (MODE == 3) {
      // software-pipelined: this iteration's DMMAs / leftovers consume the values evaluated in the previous
      // iteration; this iteration's Horner results are only needed by the next one
      double an[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double a = th[P - 1];
#pragma unroll
        for (int p = P - 2; p >= 0; --p) a = fma(a, tl[u], th[p]);
        an[u] = a;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        dmma884(acc[u][0], acc[u][1], av[u], b);
#pragma unroll
        for (int c = 0; c < REM; ++c) accx[u][c] = fma(av[u], rv[c], accx[u][c]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) av[u] = an[u];
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double a = th[P - 1];
#pragma unroll
        for (int p = P - 2; p >= 0; --p) a = vfma(a, tl[u], th[p]);
        av[u] = a;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) dmma884(acc[u][0], acc[u][1], av[u], b);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < REM; ++c) accx[u][c] = vfma(av[u], rv[c], accx[u][c]);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) th[p] += 1e-9;
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

// m16n8k16: per unit 8 A elements per lane (Horner each), one DMMA, REM leftover DFMA per element
template <int U, int P, int REM>
__global__ void __launch_bounds__(512, 1) mix16816(double* out, int iters, double t0) {
  double acc[U][4], accx[U][REM > 0 ? REM : 1];
  double th[P], tl[U], b[4], rv[REM > 0 ? REM : 1];
#pragma unroll
  for (int p = 0; p < P; ++p) th[p] = threadIdx.x * 1e-3 + p;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-5 - i * 1e-6;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0.0;
    tl[u] = t0 + u * 1e-3;
#pragma unroll
    for (int c = 0; c < (REM > 0 ? REM : 1); ++c) accx[u][c] = 0.0;
  }
#pragma unroll
  for (int c = 0; c < (REM > 0 ? REM : 1); ++c) rv[c] = 0.5 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double a[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        double v = th[P - 1] + e * 1e-7;
#pragma unroll
        for (int p = P - 2; p >= 0; --p) v = fma(v, tl[u], th[p]);
        a[e] = v;
      }
      dmma16816(acc[u], a, b);
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int c = 0; c < REM; ++c) accx[u][c] = fma(a[e], rv[c], accx[u][c]);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) th[p] += 1e-9;
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
#pragma unroll
    for (int c = 0; c < REM; ++c) s += accx[u][c];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
static float time_it(K kern, int sms, int threads, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<sms, threads>>>(out, iters, 0.3);
  cudaEventRecord(e0);
  kern<<<sms, threads>>>(out, iters, 0.3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

static void report(const char* name, float ms, double mma_mac, double dfma, int sms, int threads, int iters) {
  const double warps = (double)sms * threads / 32;
  mma_mac *= warps * iters;
  dfma *= warps * iters * 32;
  const double ideal_ms = (2 * mma_mac / 37.0e12 + 2 * dfma / 33.6e12) * 1e3;
  printf("%-40s threads=%d: %.3f ms, pipe model %.3f ms -> %.1f%%\n", name, threads, ms, ideal_ms,
         100.0 * ideal_ms / ms);
}

template <int U, int P, int REM, int MODE>
static void run884(int sms, double* out, int threads) {
  const int iters = 4000;
  float ms = time_it(mix884<U, P, REM, MODE>, sms, threads, out, iters);
  char name[64];
  snprintf(name, sizeof name, "m8n8k4 U=%d P=%d REM=%d mode=%d", U, P, REM, MODE);
  report(name, ms, 256.0 * U, (double)U * (P - 1 + REM), sms, threads, iters);
}

template <int U, int P, int REM>
static void run16816(int sms, double* out, int threads) {
  const int iters = 1000;
  float ms = time_it(mix16816<U, P, REM>, sms, threads, out, iters);
  char name[64];
  snprintf(name, sizeof name, "m16n8k16 U=%d P=%d REM=%d", U, P, REM);
  report(name, ms, 2048.0 * U, 8.0 * U * (P - 1 + REM), sms, threads, iters);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  run884<6, 1, 0, 0>(sms, out, 512);  // DMMA only
  run884<6, 3, 0, 0>(sms, out, 512);  // Horner + DMMA
  run884<6, 3, 0, 3>(sms, out, 512);
  run884<6, 1, 2, 0>(sms, out, 512);  // DMMA + leftover
  run884<6, 3, 2, 0>(sms, out, 512);
  run884<6, 3, 2, 3>(sms, out, 512);
  run884<6, 3, 2, 3>(sms, out, 256);
  run884<12, 3, 2, 3>(sms, out, 256);
  run884<12, 3, 2, 3>(sms, out, 384);
  run884<8, 3, 2, 3>(sms, out, 384);
  run884<4, 3, 2, 3>(sms, out, 512);
  run884<6, 4, 0, 0>(sms, out, 512);   // c5: degree 3, m = 16 -> 2 DMMA per element, no leftover
  run884<6, 4, 0, 3>(sms, out, 512);
  return 0;
}
