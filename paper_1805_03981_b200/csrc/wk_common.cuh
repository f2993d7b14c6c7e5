// Shared definitions for the sm_100a DG-acoustics kernels.
//
// Global state layout (identical to the reference StateVector,
// /root/reference/pkg/src/wavekernel/operator.py:33-55): FP64, element-
// contiguous (E, C=d+1, n^d), components v_1..v_d, p, direction 0 fastest.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace wk {

constexpr int kMaxN = 9;  // n = k+1 <= 9  (k <= 8)

template <int D, int N>
struct Shape {
  static constexpr int C = D + 1;
  static constexpr int NODES = D == 3 ? N * N * N : N * N;
  static constexpr int NF = D == 3 ? N * N : N;  // nodes per face
  static constexpr int EPB = NODES >= 256 ? 1 : 256 / NODES;  // elements per block
  static constexpr int TPB = ((EPB * NODES + 31) / 32) * 32;
  static constexpr int STATE = C * NODES;  // doubles per element
};

// Affine per-class geometry record (see wk_geometry in wk_abi.cu):
//   [0, D*D)              G[m][i] = d xi_m / d x_i   (reference inv_jac, mesh.py:245-262)
//   [D*D, 3*D*D)          normal[m][s][i]             (outward, own side, mesh.py:265-286)
//   [3*D*D, 3*D*D + 2*D)  fscale[m][s] = face JxW factor / det J
//   [3*D*D + 2*D]         det J
template <int D>
struct GeoLayout {
  static constexpr int G = 0;
  static constexpr int NORMAL = D * D;
  static constexpr int FSCALE = 3 * D * D;
  static constexpr int DET = 3 * D * D + 2 * D;
  static constexpr int STRIDE = 3 * D * D + 2 * D + 1;
};

// Per-element material record: inv_rho, c^2 rho, tau, inv_rho/tau  (operator.py:116-123)
constexpr int kMatStride = 4;

// Output modes of the fused affine operator kernel.
enum OutMode : int {
  OUT_MINVK = 0,   // out = M^{-1} K u
  OUT_RHS = 1,     // out = -M^{-1} K u                      (operator.py:268-272)
  OUT_LSRK = 2,    // r = a r + dt f, u_out = u + b r, f = rhs (stepping.py:196-203)
  OUT_ADERB = 3,   // out = v - M^{-1} K u  (ADER final combination, stepping.py:272-284)
};

enum Parts : int { PART_CELL = 1, PART_FACE = 2, PART_BOTH = 3 };

// Neighbour table convention (int32, (E, d, 2)):  >= 0 local element,
// -1 sound-soft wall (operator.py:217-220), <= -2 ghost face slot (-2 - g)
// in a halo buffer of shape (G, C, n^{d-1}).
__host__ __device__ inline int ghost_slot(int nbr) { return -2 - nbr; }

// FP64 tensor-core MMA (DMMA), warp-wide C(8x8) += A(8x4) B(4x8):
// A lane l = M[l>>2][l&3], B lane l = X[l&3][l>>2], C lane l = Y[l>>2][2(l&3)+{0,1}]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- checked build (-DWK_CHECK, libwk_b200_check.so; tests/test_gpu_checked.py)
// Device-side asserts on every neighbour / ghost index a kernel gathers
// through, on the element range of every tile and on the dynamic shared
// memory a kernel's layout needs: a violation prints the site and traps
// (the launch fails with cudaErrorLaunchFailure) instead of reading or
// writing out of bounds.  Compiled out of the production library.
#ifdef WK_CHECK
#define WK_ASSERT(cond)                                                                   \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("WK_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                          \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define WK_ASSERT(cond) \
  do {                  \
  } while (0)
#endif
// a neighbour code of args (an AffineArgs): element < e_total, -1, or a ghost slot < n_ghost
#define WK_CHECK_NBR(args, nb)                                                       \
  WK_ASSERT(((nb) >= 0 && (long long)(nb) < (args).e_total) || (nb) == -1 ||         \
            ((nb) <= -2 && (long long)::wk::ghost_slot(nb) < (args).n_ghost))
__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}
#define WK_CHECK_SMEM(bytes) WK_ASSERT(dyn_smem_bytes() >= (unsigned)(bytes))

}  // namespace wk

// ---- small unsigned division by a runtime divisor, without the division
// subroutine: q = umulhi(a, M), M = ceil(2^32 / b); exact for a < 2^32 / b.
namespace wk {
struct UDiv {
  unsigned m, b;
  __device__ __forceinline__ explicit UDiv(unsigned d) : m(d > 1 ? 0xFFFFFFFFu / d + 1u : 0u), b(d) {}
  __device__ __forceinline__ unsigned div(unsigned a) const { return b > 1 ? __umulhi(a, m) : a; }
};
}  // namespace wk

// ---- asynchronous copies: TMA bulk (cp.async.bulk) + mbarrier -------------
namespace wk {
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared (TMA engine); bytes % 16 == 0, 16 B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 eviction priority for the streams nobody re-reads within a stage (r / V
// in, every result out): evict_first, so that the u tiles -- whose face
// nodes the neighbours gather a whole x-y chunk of tiles later -- are what
// stays resident.  Without it the 4 streams share L2 evenly, the reuse
// distance of a z-face is ~16 KB x chunk, and the stage kernel can fall into
// a state where the z-faces miss (config 5: 15 -> 18.8 ms/step).
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes,
                                              unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, unsigned bytes,
                                              unsigned long long pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::
                   "l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
// Tile-queue claim: fetch-and-increment with a RUN-TIME wrap bound (atom.inc
// returns old and stores old >= cap ? 0 : old + 1).  With atom.add, or with
// a constant bound, ptxas warp-aggregates the atomic and its SHFL broadcast
// then waits for the result right away; the inc with a run-time cap stays a
// single ATOMG whose result is consumed only where it is used.  cap must
// exceed every value the counter reaches.
__device__ __forceinline__ unsigned atomic_claim(unsigned* p, unsigned cap) {
  unsigned old;
  asm volatile("atom.relaxed.gpu.global.inc.u32 %0, [%1], %2;\n"
               : "=r"(old)
               : "l"(p), "r"(cap)
               : "memory");
  return old;
}
// bulk prefetch global -> L2 (no shared memory, no completion); 16 B granules
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async8_u32(unsigned dst, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(gmem));
}
// 1-D bulk copy shared -> global (TMA engine), bulk-group completion
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// wait until the source smem of all but `n` most recent bulk groups has been read
template <int NPEND>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NPEND) : "memory");
}
template <int NPEND>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(NPEND) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for the phase with a suspend-time hint: the warp sleeps in hardware
// until the phase completes (or ~10 ms pass) instead of re-issuing try_wait
// in a tight loop.  Under the board power cap the polling of the waiting
// warps takes power from the working ones (measured: the direction-parallel
// stage kernel fell from 14.7 to 18.8 ms/step once the cap was reached).
#ifndef WK_MBAR_HINT
#define WK_MBAR_HINT 1
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
#if WK_MBAR_HINT
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WK_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@p bra WK_DONE;\n"
      "bra WK_WAIT;\n"
      "WK_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}
}  // namespace wk
