// Whole-run LSRK kernel for SMALL meshes (BASELINE config 1: 2-D 16^2, k = 3,
// 12 k DoF): K time steps x S stages in ONE launch of ONE thread-block
// cluster (up to 16 CTAs, one per SM) whose shared memories hold the entire
// state.
//
// At config 1 the streamed path is launch-bound: 5 persistent-kernel launches
// per step (~5 us each, even replayed from a CUDA graph) for 12 k DoF of
// work.  Here each CTA of the cluster owns a contiguous element range and
// keeps u (two buffers), r and the face integrands of its elements in
// shared memory for the whole run; a stage reads the neighbours' face values
// straight from the owning CTA's shared memory through distributed shared
// memory (cluster.map_shared_rank), and one cluster barrier per stage
// (barrier.cluster arrive/wait, release/acquire) separates the stages.  Stage
// i reads u[p] and writes u[p^1], so the barrier after it is the only
// synchronisation needed (nobody writes a buffer that is still being read).
//
// Arithmetic: identical operation order to affine_stream_kernel (wk_stream.cuh)
// on Cartesian single-class affine cells -- the same split-form collapse
// (A, L0, L1 as constant-bank operands), the same face integrand
// (cart_face_flux), the same LSRK update fma sequence -- so the result is
// BITWISE equal to the stage-by-stage path (tests/test_gpu_small.py).
#pragma once
#include <cooperative_groups.h>

#include "wk_group.cuh"

namespace wk {

constexpr int kSmallMaxCluster = 16;
constexpr int kSmallMaxStages = 16;

struct SmallArgs {
  const double* u_in;          // (E, C, NODES) initial state
  double* u_out;               // final state (may alias u_in)
  const int* nbr;              // (E, d, 2)
  const double* mat;           // (E, kMatStride)
  const double* geo;           // the single class record (GeoLayout)
  long long E;
  int epc;                     // elements per CTA
  int stages, steps, stab;
  double dt;
  double a[kSmallMaxStages], b[kSmallMaxStages];
  double cA[kMaxN * kMaxN], cL0[kMaxN], cL1[kMaxN];
};

template <int D, int N>
struct SmallCfg {
  static constexpr int C = D + 1, NODES = D == 3 ? N * N * N : N * N, NF = D == 3 ? N * N : N;
  static constexpr int TILE = C * NODES;                       // doubles per element
  // per element: u[2], r, face integrands (fv, fp per face node), 2d neighbour
  // ids (as doubles' worth of ints), material
  static constexpr int PER_EL = 3 * TILE + 2 * D * 2 * NF + D + 4;
  __host__ __device__ static size_t bytes(int epc) { return sizeof(double) * ((size_t)epc * PER_EL + GeoLayout<D>::STRIDE + 1); }
};

template <int D, int N>
__global__ void __launch_bounds__(1024) small_lsrk_kernel(const __grid_constant__ SmallArgs A) {
  namespace cg = cooperative_groups;
  using K = SmallCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, TILE = K::TILE;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double smem[];
  const int epc = A.epc;
  const int rank = (int)cluster.block_rank();
  const long long e_lo = (long long)rank * epc;
  const int nel = (int)max(0LL, min((long long)epc, A.E - e_lo));
  double* const ub0 = smem;
  double* const ub1 = ub0 + (size_t)epc * TILE;
  double* const sr = ub1 + (size_t)epc * TILE;
  double* const sF = sr + (size_t)epc * TILE;                   // [el][f][fv|fp][fn]
  double* const smat = sF + (size_t)epc * 2 * D * 2 * NF;
  int* const snbr = reinterpret_cast<int*>(smat + (size_t)epc * 4);
  double* const geo = reinterpret_cast<double*>(snbr) + (size_t)epc * D;
  const int tid = threadIdx.x, nth = blockDim.x;
  WK_CHECK_SMEM(K::bytes(epc));

  for (int i = tid; i < GLy::STRIDE; i += nth) geo[i] = A.geo[i];
  for (int i = tid; i < nel * TILE; i += nth) ub0[i] = A.u_in[e_lo * TILE + i];
  for (int i = tid; i < nel * 4; i += nth) smat[i] = A.mat[e_lo * kMatStride + i];
  for (int i = tid; i < nel * 2 * D; i += nth) {
    const int nb = A.nbr[e_lo * 2 * D + i];
    WK_ASSERT(nb >= -1 && nb < A.E);
    snbr[i] = nb;
  }
  cluster.sync();

  int par = 0;
  for (int step = 0; step < A.steps; ++step) {
    for (int st = 0; st < A.stages; ++st) {
      const double* const cur = par ? ub1 : ub0;
      double* const nxt = par ? ub0 : ub1;
      const double a = A.a[st], b = A.b[st];
      // ---- face integrands u_hat - F_n(own)/2 at every face node (operator.py:217-239)
      for (int t = tid; t < nel * 2 * D * NF; t += nth) {
        const int fn = t % NF, ef = t / NF;
        const int f = ef % (2 * D), el = ef / (2 * D);
        const int m = f >> 1, s = f & 1;
        const double* mt = smat + el * 4;
        const double ir = mt[0], c2r = mt[1], tau = mt[2], irt = mt[3];
        const int on = face_to_node<N>(m, s, fn);
        const double vo = cur[(el * C + m) * NODES + on];
        const double po = cur[(el * C + D) * NODES + on];
        const int nb = snbr[el * 2 * D + f];
        double vx, px;
        if (nb == -1) {                       // sound-soft mirror (operator.py:217-220)
          vx = vo;
          px = -po;
        } else {                              // the neighbour's trace, from its CTA
          const int owner = nb / epc, li = nb - owner * epc;
          const double* rem = cluster.map_shared_rank(const_cast<double*>(cur), owner) +
                              (size_t)li * TILE;
          const int nn = face_to_node<N>(m, 1 - s, fn);
          vx = rem[m * NODES + nn];
          px = rem[D * NODES + nn];
        }
        double fv, fp;
        cart_face_flux(vo, po, vx, px, geo[GLy::NORMAL + (m * 2 + s) * D + m],
                       geo[GLy::FSCALE + m * 2 + s], ir, c2r, tau, irt, A.stab != 0, fv, fp);
        double* F = sF + ((size_t)(el * 2 * D + f) * 2) * NF + fn;
        F[0] = fv;
        F[NF] = fp;
      }
      __syncthreads();
      // ---- M^{-1} K u at every node and the LSRK update (wk_stream.cuh order)
      for (int t = tid; t < nel * NODES; t += nth) {
        const int el = t / NODES, node = t - el * NODES;
        const double* mt = smat + el * 4;
        const double ir = mt[0], c2r = mt[1];
        const double* ue = cur + (size_t)el * TILE;
        double* ne = nxt + (size_t)el * TILE;
        double* re = sr + (size_t)el * TILE;
        double pacc = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
          const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
          const int im = (node / sm) % N;
          const int base = node - im * sm;
          double ap = 0.0, av = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const double aa = A.cA[im * N + j];
            ap = fma(aa, ue[D * NODES + base + j * sm], ap);
            av = fma(aa, ue[m * NODES + base + j * sm], av);
          }
          const int fn = node_to_face<N>(m, node);
          const double* F0 = sF + ((size_t)(el * 2 * D + 2 * m) * 2) * NF + fn;
          const double* F1 = F0 + 2 * NF;
          const double l0 = A.cL0[im], l1 = A.cL1[im];
          const double gmm = geo[m * D + m];
          const double resv = fma(ir * gmm, ap, fma(l0, F0[0], l1 * F1[0]));
          double resp = fma(c2r * gmm, av, fma(l0, F0[NF], l1 * F1[NF]));
          if (m > 0) resp += pacc;
          pacc = resp;
          const int iv = m * NODES + node;
          const double fr = -resv * A.dt;
          const double rr = a != 0.0 ? fma(a, re[iv], fr) : fr;
          re[iv] = rr;
          ne[iv] = fma(b, rr, ue[iv]);
        }
        const int ip = D * NODES + node;
        const double fr = -pacc * A.dt;
        const double rr = a != 0.0 ? fma(a, re[ip], fr) : fr;
        re[ip] = rr;
        ne[ip] = fma(b, rr, ue[ip]);
      }
      cluster.sync();          // stage done everywhere: its input buffer is free
      par ^= 1;
    }
  }
  const double* fin = par ? ub1 : ub0;
  for (int i = tid; i < nel * TILE; i += nth) A.u_out[e_lo * TILE + i] = fin[i];
}

}  // namespace wk
