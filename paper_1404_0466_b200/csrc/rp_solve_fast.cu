// Specialised instantiations of the fused eval+solve for the output counts / degrees of the
// BASELINE configs: m = 1 (c1), m = 10 (c2-c4, degree 2), m = 16 (c5, degree 3). They run the
// warp-specialised kernel (rp_solve_ws.cuh) with the deepest stage ring that fits shared memory
// in each direction when RP_SOLVE_WS=1; by default they run the 16-warp cp.async kernel
// (rp_solve.cuh).
#include <cstdlib>

#include "rp_solve_ws.cuh"

#ifndef RP_SOLVE_LG
#define RP_SOLVE_LG 4
#endif

namespace rp {

// The warp-specialised kernel is opt-in (RP_SOLVE_WS=1): with 9 warps per CTA the register file
// caps it at 168 registers and it measured slower (49 ms vs 40 ms at c4) than the 16-warp
// cp.async kernel.
static const bool g_solve_ws = [] {
  const char* e = getenv("RP_SOLVE_WS");
  return e && e[0] == '1';
}();

#define RP_FAST_LIST(X) \
  X(1, 3, 16) X(1, 3, 8) X(10, 3, 2) X(10, 3, 4) X(10, 3, 8) X(10, 3, 10) X(10, 3, 12) X(10, 3, 16) X(16, 4, 4) X(16, 4, 6) \
      X(16, 4, 8)

bool has_solve_fast(int m, int P, int lam) {
#define RP_HAS(M, PP, L) \
  if (m == M && P == PP && lam == L) return true;
  RP_FAST_LIST(RP_HAS)
#undef RP_HAS
  return false;
}

template <int M, int P, int LC, bool BWD>
static int ws_pass(const SolveArgs& a, int grid, cudaStream_t st, size_t maxsmem) {
  constexpr int NT = M / 8, REM = M % 8;
  if (sizeof(double) * solve_ws_smem_doubles<P, 4, BWD>(a.S) <= maxsmem)
    return launch_solve_ws_pass<NT, REM, P, LC, 4, BWD>(a, grid, st);
  if (sizeof(double) * solve_ws_smem_doubles<P, 3, BWD>(a.S) <= maxsmem)
    return launch_solve_ws_pass<NT, REM, P, LC, 3, BWD>(a, grid, st);
  return launch_solve_ws_pass<NT, REM, P, LC, 2, BWD>(a, grid, st);
}

template <int M, int P, int LC>
static int launch_fast(const SolveArgs& a, int grid, size_t smem, cudaStream_t st) {
  if (!g_solve_ws) {
    // 16 warps (4 row groups x 4 lambda groups): measured best of 8/12/16/24/32 warps at c4.
    // A 4-stage ring (two slabs per barrier) when it fits in shared memory.
    int dev = 0, maxsm = 227 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t sm4 = solve_smem_bytes(LC, M, P, 4);
    if (sm4 <= (size_t)maxsm && !getenv("RP_SOLVE_STG3"))
      return launch_solve<M / 8, M % 8, P, LC, RP_SOLVE_LG, 4>(a, grid, sm4, st);
    return launch_solve<M / 8, M % 8, P, LC, RP_SOLVE_LG, 3>(a, grid, smem, st);
  }
  int dev = 0, maxsmem = 227 * 1024;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int rc = ws_pass<M, P, LC, false>(a, grid, st, (size_t)maxsmem);
  if (rc) return rc;
  return ws_pass<M, P, LC, true>(a, grid, st, (size_t)maxsmem);
}

int launch_solve_fast(int m, int P, int lam, const SolveArgs& a, int grid, size_t smem, cudaStream_t st) {
#define RP_LAUNCH(M, PP, L) \
  if (m == M && P == PP && lam == L) return launch_fast<M, PP, L>(a, grid, smem, st);
  RP_FAST_LIST(RP_LAUNCH)
#undef RP_LAUNCH
  return -2;
}

}  // namespace rp
