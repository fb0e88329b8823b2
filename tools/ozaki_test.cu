// Standalone check of the Ozaki-scheme int8 tcgen05 Gram (csrc/rp_ozaki.cuh) against a CPU
// long-double Gram, plus its timing at the c4 block size. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ozaki_test tools/ozaki_test.cu
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <random>
#include <vector>

#include "../paper_1404_0466_b200/csrc/rp_ozaki.cuh"

namespace rp {
int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fprintf(stderr, "\n");
  return code;
}
void count_launch() {}
bool prof_on() { return false; }
cudaEvent_t prof_event() { return nullptr; }
void prof_push(const char*, cudaEvent_t, cudaEvent_t, cudaStream_t) {}
}  // namespace rp

static int run(int nblocks, int rows, int d, bool full_check, int reps) {
  const size_t n = (size_t)nblocks * rows;
  std::vector<double> X(n * d);
  std::mt19937_64 gen(12345);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (size_t r = 0; r < n; ++r)
    for (int j = 0; j < d; ++j) X[r * d + j] = nd(gen) / std::sqrt(1.0 + j);
  double *dX, *dG;
  void* work;
  const size_t wb = rp::oz_workspace_bytes(d, rows, nblocks);
  const rp::OzIn in{nullptr, d, (int64_t)rows * d, rows, d, nblocks};
  cudaMalloc(&dX, X.size() * 8);
  cudaMalloc(&dG, (size_t)nblocks * d * d * 8);
  cudaMalloc(&work, wb);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(dG, 0, (size_t)nblocks * d * d * 8);
  rp::OzIn oin = in;
  oin.A = dX;
  int rc = rp::oz_syrk(oin, dG, d, (int64_t)d * d, false, work, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("nblocks=%d rows=%d d=%d: rc=%d sync=%s\n", nblocks, rows, d, rc, cudaGetErrorString(e));
  if (rc || e != cudaSuccess) return 1;
  std::vector<double> G((size_t)nblocks * d * d);
  cudaMemcpy(G.data(), dG, G.size() * 8, cudaMemcpyDeviceToHost);
  // check: all (i >= j) entries for small, a sample for large
  double maxabs_err = 0.0, scale = 0.0;
  std::uniform_int_distribution<int> ui(0, d - 1);
  const int nchk = full_check ? -1 : 2000;
  for (int b = 0; b < nblocks; ++b) {
    auto ref = [&](int i, int j) {
      long double s = 0;
      for (int k = 0; k < rows; ++k) s += (long double)X[((size_t)b * rows + k) * d + i] * X[((size_t)b * rows + k) * d + j];
      return (double)s;
    };
    auto check = [&](int i, int j) {
      const double r = ref(i, j), g = G[(size_t)b * d * d + (size_t)j * d + i];
      const double nrm = std::sqrt(ref(i, i) * ref(j, j));
      maxabs_err = std::fmax(maxabs_err, std::fabs(g - r) / nrm);
      scale = std::fmax(scale, nrm);
    };
    if (full_check) {
      for (int j = 0; j < d; ++j)
        for (int i = j; i < d; ++i) check(i, j);
    } else {
      for (int t = 0; t < nchk; ++t) {
        int i = ui(gen), j = ui(gen);
        if (i < j) std::swap(i, j);
        check(i, j);
      }
    }
  }
  printf("  max |G - G_ref| / sqrt(G_ii G_jj) = %.3e\n", maxabs_err);
  if (reps > 0) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    rp::oz_syrk(oin, dG, d, (int64_t)d * d, false, work, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) rp::oz_syrk(oin, dG, d, (int64_t)d * d, false, work, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double flops = (double)n * d * (d + 1);
    printf("  %.3f ms per Gram (all blocks): %.1f FP64-equivalent TFLOP/s\n", ms, flops / ms / 1e9);
  }
  cudaFree(dX);
  cudaFree(dG);
  cudaFree(work);
  return maxabs_err < 1e-12 ? 0 : 2;
}

// int8 tensor peak on this part: one CTA per SM issues back-to-back tcgen05.mma kind::i8 from the
// same shared-memory operands (no loads), N = 64 (the Ozaki kernel's shape) and N = 256.
template <int N>
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + N) * 32; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    rp::mbar_init(&bar, 1);
    rp::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(rp::smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  rp::oz_fence_before();
  __syncthreads();
  rp::oz_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = rp::smem_u32(sm), sb = sa + 128 * 32;
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    for (int it = 0; it < iters; ++it) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(rp::oz_desc_sw32(sa)), "l"(rp::oz_desc_sw32(sb)), "r"(idesc), "r"(it > 0 ? 1u : 0u));
    }
    rp::oz_commit(&bar);
    rp::mbar_wait(&bar, 0);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int N>
static void peak(int sms) {
  int* out;
  cudaMalloc(&out, sms * sizeof(int));
  const int iters = 20000;
  const size_t smem = 1024 + (128 + N) * 32;
  i8_peak_kernel<N><<<sms, 128, smem>>>(100, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  i8_peak_kernel<N><<<sms, 128, smem>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 128 * N * 32 * (double)iters * sms;
  printf("int8 tcgen05 peak, M=128 N=%d K=32: %.1f TOPS (%s)\n", N, ops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

// Trailing-update shapes of the blocked Cholesky: C_b -= A_b A_b^T with A_b = the M x K panel
// below the diagonal inside a d x d column-major matrix (lda = d), nbatch matrices.
static void trailing(int d, int M, int K, int nbatch, int reps) {
  double *dA, *dC;
  const size_t nn = (size_t)nbatch * d * d;
  cudaMalloc(&dA, nn * 8);
  cudaMalloc(&dC, nn * 8);
  std::vector<double> h((size_t)d * d);
  std::mt19937_64 gen(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (auto& v : h) v = nd(gen);
  for (int b = 0; b < nbatch; ++b) cudaMemcpy(dA + (size_t)b * d * d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, nn * 8);
  const rp::OzIn in{dA + (d - M), d, (int64_t)d * d, K, M, nbatch};
  void* work;
  cudaMalloc(&work, rp::oz_workspace_bytes(M, K, nbatch));
  double* C = dC + (size_t)(d - M) * d + (d - M);
  rp::oz_syrk(in, C, d, (int64_t)d * d, true, work, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) rp::oz_syrk(in, C, d, (int64_t)d * d, true, work, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double flops = (double)nbatch * M * (M + 128.0) * K;  // lower 128-tiles incl. diagonal tiles
  printf("trailing M=%d K=%d batch=%d: %.3f ms, %.1f FP64-equivalent TFLOP/s (%s)\n", M, K, nbatch, ms,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(dA);
  cudaFree(dC);
  cudaFree(work);
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 't') {
    const int shapes[][3] = {{2560, 1536, 10}, {1024, 1536, 10}, {2560, 1536, 40}, {3072, 1024, 10},
                             {3584, 512, 10}, {3584, 512, 40}, {2048, 2048, 10}, {3328, 768, 10}};
    for (auto& sh : shapes) trailing(4096, sh[0], sh[1], sh[2], 5);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'p') {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    peak<64>(sms);
    peak<128>(sms);
    peak<256>(sms);
    return 0;
  }
  int rc = 0;
  rc |= run(2, 1000, 256, true, 0);
  rc |= run(1, 40000, 128, true, 0);  // K chunking (kchunk < kpad)
  if (argc > 1) rc |= run(8, 12500, 4096, false, 3);
  printf("rc=%d\n", rc);
  return rc;
}
