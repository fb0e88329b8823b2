// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64) throughput,
// and the two issued concurrently. Used to set the FP64 roofline denominator
// (MEASURED_PEAKS.json has only HBM and bf16). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks tools/fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int ACC>
__global__ void dmma_kernel(double* out, int iters) {
  double c[ACC][2];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma884(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma16816(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
               "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int ACC>
__global__ void dmma16816_kernel(double* out, int iters) {
  double c[ACC][4];
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 - i;
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma16816(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// DMMA and DFMA interleaved in the same warp: does the eval (DFMA) hide under DMMA?
template <int ACC, int NF>
__global__ void mixed_kernel(double* out, int iters, double x, double y) {
  double c[ACC][2];
  double f[NF];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma884(c[i][0], c[i][1], a, b);
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  printf("{\"sms\": %d", sms);
  for (int blocksPerSM : {1, 2, 4}) {
    int threads = 256, iters = 20000;
    dim3 grid(sms * blocksPerSM);
    for (int w = 0; w < 2; ++w) dfma_kernel<16><<<grid, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_kernel<16><<<grid, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)threads * grid.x;
    printf(", \"dfma_tflops_b%d\": %.3f", blocksPerSM, flops / ms / 1e9);
  }
  for (int blocksPerSM : {1, 2, 4}) {
    int threads = 256, iters = 4000;
    dim3 grid(sms * blocksPerSM);
    for (int w = 0; w < 2; ++w) dmma_kernel<8><<<grid, threads>>>(out, iters);
    cudaEventRecord(e0);
    dmma_kernel<8><<<grid, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * iters * (double)(threads / 32) * grid.x;
    printf(", \"dmma884_tflops_b%d\": %.3f", blocksPerSM, flops / ms / 1e9);
  }
  for (int blocksPerSM : {1, 2}) {
    int threads = 256, iters = 1000;
    dim3 grid(sms * blocksPerSM);
    for (int w = 0; w < 2; ++w) dmma16816_kernel<4><<<grid, threads>>>(out, iters);
    cudaEventRecord(e0);
    dmma16816_kernel<4><<<grid, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 4 * iters * (double)(threads / 32) * grid.x;
    printf(", \"dmma16816_tflops_b%d\": %.3f", blocksPerSM, flops / ms / 1e9);
  }
  {
    int threads = 256, iters = 4000;
    dim3 grid(sms * 2);
    for (int w = 0; w < 2; ++w) mixed_kernel<8, 8><<<grid, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    mixed_kernel<8, 8><<<grid, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double mma_flops = 2.0 * 256 * 8 * iters * (double)(threads / 32) * grid.x;
    double fma_flops = 2.0 * 8 * iters * (double)threads * grid.x;
    printf(", \"mixed_ms\": %.3f, \"mixed_mma_tflops\": %.3f, \"mixed_dfma_tflops\": %.3f", ms,
           mma_flops / ms / 1e9, fma_flops / ms / 1e9);
  }
  {
    size_t n = (size_t)1 << 27;  // 2 GiB per buffer of double2? no: 2^27 * 16 B = 2 GiB
    double2 *a, *b;
    CK(cudaMalloc(&a, n * sizeof(double2)));
    CK(cudaMalloc(&b, n * sizeof(double2)));
    cudaMemset(a, 0, n * sizeof(double2));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf(", \"copy_gbs\": %.1f", 2.0 * n * sizeof(double2) / best / 1e6);
  }
  printf("}\n");
  return 0;
}
