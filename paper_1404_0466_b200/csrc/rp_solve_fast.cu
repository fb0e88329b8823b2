// Specialised instantiations of the fused eval+solve for the output counts / degrees of the
// BASELINE configs: m = 1 (c1), m = 10 (c2-c4, degree 2), m = 16 (c5, degree 3), each with the
// lambda chunks the planner (rp_solve.cu) can pick (c5: 7-lambda chunks fill 3.9 waves of CTAs where
// 8-lambda chunks leave the 4th wave 40% occupied). Every entry is exercised against the oracle by
// tests/test_gpu_kernels.py::test_every_solve_instantiation (rp_set_option("solve_lam", n)).
#include "rp_solve.cuh"

// Lambda groups of warps (each warp: 16 rows x ceil(LC / LG) lambdas). Large chunks: 12 warps (measured at
// c4 in round 2: 30.5-30.9 ms for both passes vs 31.9-32.2 with 16 warps and 33+ with a producer warp added;
// c5 408 vs 413 ms).
#ifndef RP_SOLVE_LG
#define RP_SOLVE_LG 3
#endif

namespace rp {

#define RP_FAST_LIST(X) \
  X(1, 3, 16) X(1, 3, 8) X(10, 3, 2) X(10, 3, 3) X(10, 3, 4) X(10, 3, 6) X(10, 3, 8) X(10, 3, 9) X(10, 3, 10) X(10, 3, 11) \
      X(10, 3, 12) X(10, 3, 16) X(16, 4, 4) X(16, 4, 6) X(16, 4, 7) X(16, 4, 8)

bool has_solve_fast(int m, int P, int lam) {
#define RP_HAS(M, PP, L) \
  if (m == M && P == PP && lam == L) return true;
  RP_FAST_LIST(RP_HAS)
#undef RP_HAS
  return false;
}

// Ring depth:
// small chunks (<= 4 lambdas: little arithmetic per slab, e.g. the one-fold-per-GPU case) are bound by
// the copy latency and get a 6-stage ring with 4 slabs in flight when it fits; otherwise a 4-stage ring
// (two slabs in flight) when it fits, else 3 stages.
template <int M, int P, int LC>
static int stages_fast() {
  int dev = 0, maxsm = 227 * 1024;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (LC <= 4 && solve_smem_max(LC, M, P, 6) <= (size_t)maxsm) return 6;
  return solve_smem_max(LC, M, P, 4) <= (size_t)maxsm ? 4 : 3;
}

// lambda groups of warps for a chunk of LC lambdas: 8 warps for small chunks (every warp has a lambda;
// one fold per GPU, tools/solve_nf.py: 14.4 -> 12.9 ms with 2-lambda chunks; 4 warps: 13.5 ms)
template <int LC>
constexpr int lg_for() {
  return LC <= 4 ? 2 : RP_SOLVE_LG;
}

template <int M, int P, int LC>
static int launch_fast(const SolveArgs& a, int grid, cudaStream_t st, bool tail) {
  constexpr int LG = lg_for<LC>();
  switch (stages_fast<M, P, LC>()) {
    case 6: return launch_solve<M / 8, M % 8, P, LC, LG, (LC <= 4 ? 6 : 4)>(a, grid, st, tail);
    case 4: return launch_solve<M / 8, M % 8, P, LC, LG, 4>(a, grid, st, tail);
    default: return launch_solve<M / 8, M % 8, P, LC, LG, 3>(a, grid, st, tail);
  }
}

template <int M, int P, int LC>
static int clusters_fast(int cl) {
  constexpr int LG = lg_for<LC>();
  switch (stages_fast<M, P, LC>()) {
    case 6: return solve_clusters<M / 8, M % 8, P, LC, LG, (LC <= 4 ? 6 : 4)>(LC, M, P, cl);
    case 4: return solve_clusters<M / 8, M % 8, P, LC, LG, 4>(LC, M, P, cl);
    default: return solve_clusters<M / 8, M % 8, P, LC, LG, 3>(LC, M, P, cl);
  }
}

int solve_fast_clusters(int m, int P, int lam, int cl) {
#define RP_CL(M, PP, L) \
  if (m == M && P == PP && lam == L) return clusters_fast<M, PP, L>(cl);
  RP_FAST_LIST(RP_CL)
#undef RP_CL
  return 0;
}

int launch_solve_fast(int m, int P, int lam, const SolveArgs& a, int grid, cudaStream_t st, bool tail) {
#define RP_LAUNCH(M, PP, L) \
  if (m == M && P == PP && lam == L) return launch_fast<M, PP, L>(a, grid, st, tail);
  RP_FAST_LIST(RP_LAUNCH)
#undef RP_LAUNCH
  return -2;
}

}  // namespace rp
