// (5) Fused evaluate + solve: host dispatch of rp_eval_solve and the generic (runtime P and
// chunk size) kernel instantiations. The kernel itself is in rp_solve.cuh; the specialised
// (compile-time P and chunk) instantiations used by the BASELINE configs are in rp_solve_fast.cu.
#include "rp_solve.cuh"
#include "../../include/ridgepath_b200.h"

using namespace rp;

static int launch_generic(int m, const SolveArgs& a, int grid, size_t smem, cudaStream_t st) {
  switch (m) {
    case 1: return launch_solve<0, 1, 0, 0>(a, grid, smem, st);
    case 2: return launch_solve<0, 2, 0, 0>(a, grid, smem, st);
    case 3: return launch_solve<0, 3, 0, 0>(a, grid, smem, st);
    case 4: return launch_solve<0, 4, 0, 0>(a, grid, smem, st);
    case 5: return launch_solve<0, 5, 0, 0>(a, grid, smem, st);
    case 6: return launch_solve<0, 6, 0, 0>(a, grid, smem, st);
    case 7: return launch_solve<0, 7, 0, 0>(a, grid, smem, st);
    case 8: return launch_solve<1, 0, 0, 0>(a, grid, smem, st);
    case 9: return launch_solve<1, 1, 0, 0>(a, grid, smem, st);
    case 10: return launch_solve<1, 2, 0, 0>(a, grid, smem, st);
    case 11: return launch_solve<1, 3, 0, 0>(a, grid, smem, st);
    case 12: return launch_solve<1, 4, 0, 0>(a, grid, smem, st);
    case 13: return launch_solve<1, 5, 0, 0>(a, grid, smem, st);
    case 14: return launch_solve<1, 6, 0, 0>(a, grid, smem, st);
    case 15: return launch_solve<1, 7, 0, 0>(a, grid, smem, st);
    default: return launch_solve<2, 0, 0, 0>(a, grid, smem, st);
  }
}

extern "C" int rp_eval_solve(const double* theta, int d, int r, int nf, const double* rhs, int m,
                             const double* tvals, int q, double* W, int64_t ldw, int* flags, void* stream) {
  RP_REQUIRE(d >= 1 && nf >= 1 && q >= 1, "rp_eval_solve: bad sizes d=%d nf=%d q=%d", d, nf, q);
  RP_REQUIRE(r >= 0 && r + 1 <= SOLVE_PMAX, "rp_eval_solve: degree %d outside [0, %d]", r, SOLVE_PMAX - 1);
  RP_REQUIRE(m >= 1 && m <= 16, "rp_eval_solve: %d outputs per call (max 16)", m);
  RP_REQUIRE(ldw >= (int64_t)q * m && ldw % 2 == 0, "rp_eval_solve: ldw=%lld must be even and >= q*m",
             (long long)ldw);
  RP_REQUIRE(((uintptr_t)theta & 15) == 0 && ((uintptr_t)W & 15) == 0, "rp_eval_solve: 16-byte alignment");
  cudaStream_t st = (cudaStream_t)stream;
  const int P = r + 1;
  const int nt = (d + 63) / 64;
  int dev = 0, sms = 148, maxsmem = 227 * 1024;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // Candidate chunk sizes: specialised kernels (full chunks, compile-time P) and the generic
  // kernel; pick the lowest (waves x chunk) cost, weighting the generic kernel's overhead.
  int best_lam = 0;
  bool best_fast = false;
  double best_cost = 1e300;
  for (int lam = SOLVE_LC; lam >= 1; --lam) {
    if (lam * m > 256) continue;  // one thread per (lambda, output) column in the diagonal solve
    if (solve_smem_bytes(lam, m, P) > (size_t)maxsmem) continue;
    const int chunks = (q + lam - 1) / lam;
    const long long ctas = (long long)nf * chunks;
    const double waves = (double)((ctas + sms - 1) / sms);
    const double base = waves * lam * (1.0 + 0.02 * (SOLVE_LC - lam));
    const bool fast_ok = q >= lam && has_solve_fast(m, P, lam) && ((m % 2 == 0) || ((q - lam) % 2 == 0));
    const bool gen_ok = lam <= SOLVE_LC_GENERIC && !((m & 1) && (lam & 1) && q > 1);  // odd m: even chunks
    if (fast_ok && base < best_cost - 1e-9) {
      best_cost = base;
      best_lam = lam;
      best_fast = true;
    }
    if (gen_ok && 2.5 * base < best_cost - 1e-9) {
      best_cost = 2.5 * base;
      best_lam = lam;
      best_fast = false;
    }
  }
  RP_REQUIRE(best_lam >= 1, "rp_eval_solve: no chunk size fits shared memory");
  SolveArgs a;
  a.theta = theta;
  a.theta_fold_stride = rp_tile_count(d) * P * 4096;
  a.rhs = rhs;
  a.rhs_fold_stride = (int64_t)nt * 64 * m;
  a.W = W;
  a.ldw = ldw;
  a.w_fold_stride = (int64_t)nt * 64 * ldw;
  a.tvals = tvals;
  a.flags = flags;
  a.q = q;
  a.m = m;
  a.d = d;
  a.nt = nt;
  a.P = P;
  a.lam_per_cta = best_lam;
  a.chunks = (q + best_lam - 1) / best_lam;
  a.S = solve_stride(best_lam, m);
  const size_t smem = solve_smem_bytes(best_lam, m, P);
  const int grid = nf * a.chunks;
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)nf * q, st);
  if (e != cudaSuccess) return cuda_status(e, "rp_eval_solve memset");
  if (best_fast) return launch_solve_fast(m, P, best_lam, a, grid, smem, st);
  return launch_generic(m, a, grid, smem, st);
}
