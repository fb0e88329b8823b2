// Microbenchmark (experiments only): read bandwidth of 5 concurrent streams whose base addresses are a
// fixed stride apart (the fit kernel reads the s factor matrices at d*d*8 = 2^27-byte strides at c4).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read5(const double2* base, long long stride2, long long n2, double* out) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    double2 a = __ldcs(base + i), b = __ldcs(base + stride2 + i), c = __ldcs(base + 2 * stride2 + i),
            d = __ldcs(base + 3 * stride2 + i), e = __ldcs(base + 4 * stride2 + i);
    acc += a.x + b.x + c.x + d.x + e.x + a.y + b.y + c.y + d.y + e.y;
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const long long n = 1ll << 24;  // doubles per stream (128 MB)
  double* buf;
  cudaMalloc(&buf, (size_t)(5 * (n + (1 << 20))) * 8);
  cudaMemset(buf, 0, (size_t)(5 * (n + (1 << 20))) * 8);
  double* out;
  cudaMalloc(&out, 8);
  long long pads[] = {0, 64, 512, 4096, 65536, 262144};
  for (long long pad : pads) {
    const long long stride = n + pad;  // doubles
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    read5<<<148 * 8, 256>>>((const double2*)buf, stride / 2, n / 2, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) read5<<<148 * 8, 256>>>((const double2*)buf, stride / 2, n / 2, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stride = 2^27 B + %lld B: %.0f GB/s\n", pad * 8, 5.0 * 5 * n * 8 / (ms / 1e3) / 1e9);
  }
  return 0;
}
