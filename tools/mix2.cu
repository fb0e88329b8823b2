// Microbenchmark (experiments only): how the FP64 pipe handles the eval+solve instruction mix
// (Horner DFMA -> DMMA + leftover DFMA) depending on instruction order and MMA shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix2 tools/mix2.cu
#include <cstdio>
#include <cstdlib>
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
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(err));
    exit(1);
  }
  float ms = 0.f;
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


// MODE-4 kernel: the solve's per-warp k-step structure with operands from shared memory: 2 m-tiles with
// their own P coefficient values (one 16-byte load per plane), LH lambdas each with its own B value and
// REM leftover values (loaded per k-step), Horner per (lambda, m-tile), DMMA + REM DFMA.
template <int LH, int P, int REM, bool LOADS>
__global__ void __launch_bounds__(512, 1) mixreal(double* out, int iters, double t0) {
  __shared__ __align__(16) double sm[6000];
  for (int i = threadIdx.x; i < 6000; i += blockDim.x) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[LH][2][2], accx[LH][2][REM > 0 ? REM : 1], tl[LH];
#pragma unroll
  for (int i = 0; i < LH; ++i) {
    tl[i] = t0 + i * 1e-3;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      acc[i][mt][0] = acc[i][mt][1] = 0.0;
#pragma unroll
      for (int c = 0; c < (REM > 0 ? REM : 1); ++c) accx[i][mt][c] = 0.0;
    }
  }
  double thr[2][P], br[LH], rvr[LH][REM > 0 ? REM : 1];
#pragma unroll
  for (int p = 0; p < P; ++p) thr[0][p] = thr[1][p] = 0.5 + p;
#pragma unroll
  for (int i = 0; i < LH; ++i) {
    br[i] = 1.0 + i;
#pragma unroll
    for (int c = 0; c < (REM > 0 ? REM : 1); ++c) rvr[i][c] = 0.25 + c;
  }
  for (int it = 0; it < iters; ++it) {
    const int ks = it & 3;
    double th[2][P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (LOADS) {
        const double2 v = *reinterpret_cast<const double2*>(sm + p * 1088 + (ks * 4 + t) * 68 + 2 * g);
        th[0][p] = v.x;
        th[1][p] = v.y;
      } else {
        th[0][p] = thr[0][p] + it * 1e-12;
        th[1][p] = thr[1][p] + it * 1e-12;
      }
    }
    const double* wrow = sm + 3264 + (ks * 4 + t) * 124;
#pragma unroll
    for (int i = 0; i < LH; ++i) {
      double b, rv[REM > 0 ? REM : 1];
      if (LOADS) {
        b = wrow[i * 10 + g];
        if (REM == 2) {
          const double2 v2 = *reinterpret_cast<const double2*>(wrow + i * 10 + 8);
          rv[0] = v2.x;
          rv[REM > 1 ? 1 : 0] = v2.y;
        }
      } else {
        b = br[i];
#pragma unroll
        for (int c = 0; c < REM; ++c) rv[c] = rvr[i][c];
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        double av = th[mt][P - 1];
#pragma unroll
        for (int p = P - 2; p >= 0; --p) av = fma(av, tl[i], th[mt][p]);
        dmma884(acc[i][mt][0], acc[i][mt][1], av, b);
#pragma unroll
        for (int c = 0; c < REM; ++c) accx[i][mt][c] = fma(av, rv[c], accx[i][mt][c]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < LH; ++i)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      s += acc[i][mt][0] + acc[i][mt][1];
#pragma unroll
      for (int c = 0; c < REM; ++c) s += accx[i][mt][c];
    }
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int LH, int P, int REM, bool LOADS>
static void runreal(int sms, double* out, int threads) {
  const int iters = 4000;
  float ms = time_it(mixreal<LH, P, REM, LOADS>, sms, threads, out, iters);
  char name[64];
  snprintf(name, sizeof name, "real LH=%d P=%d REM=%d loads=%d", LH, P, REM, (int)LOADS);
  report(name, ms, 256.0 * 2 * LH, 2.0 * LH * (P - 1 + REM), sms, threads, iters);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  run884<6, 3, 2, 0>(sms, out, 512);
  runreal<3, 3, 2, false>(sms, out, 512);
  runreal<3, 3, 2, true>(sms, out, 512);
  runreal<6, 3, 2, true>(sms, out, 256);
  runreal<3, 3, 2, true>(sms, out, 256);
  return 0;
}
