// Warp-group fused operator for axis-aligned (Cartesian) affine cells — the
// hot path of BASELINE configs 1, 2, 4 and 5 (LSRK stage, rhs, M^{-1}K,
// ADER final combination).
//
// Arithmetic: wk_affine.cuh's collapsed split form specialised to diagonal
// G (see wk_pencil.cuh for the derivation):
//   v_m  <- ir G_mm A_m p   + L0 (x) Fv_{m,0} + L1 (x) Fv_{m,1}     (direction m only)
//   p    <- sum_m c2r G_mm A_m v_m + L0 (x) Fp_{m,0} + L1 (x) Fp_{m,1}
//
// Mapping: a GROUP of 32 (or 64/96) threads owns EPG elements.  No CTA-wide
// barriers: each group synchronises with __syncwarp / its own named barrier,
// so every resident warp is an independent stream of element work and the
// SM overlaps one group's global loads with another's arithmetic.
//   1. cp.async the u tile and the neighbour face-node values (only the v_m
//      and p components are needed on a Cartesian face: half the halo bytes);
//   2. face integrands, in place;
//   3. for m = 0..d-1: lane = pencil along m.  It loads the p- and v_m-lines
//      (n loads for 2 n^2 FMAs), reads r / V for its nodes straight from
//      global, finishes v_m (update + store) and accumulates its share of p
//      in shared memory; the last direction finishes p.
#pragma once
#include "wk_stage.cuh"

namespace wk {

template <int D, int N>
struct GroupCfg {
  static constexpr int C = D + 1;
  static constexpr int NODES = D == 3 ? N * N * N : N * N;
  static constexpr int NF = D == 3 ? N * N : N;
  static constexpr int EPG = NF >= 32 ? 1 : 32 / NF;               // elements per group
  static constexpr int TG = ((EPG * NF + 31) / 32) * 32;           // threads per group
  static constexpr int GPB = TG >= 128 ? 1 : 128 / TG;             // groups per block
  static constexpr int TPB = TG * GPB;
  // per-group smem (doubles): u tile | r (or V) tile | p partial sums
  static constexpr int G_U = 0;
  static constexpr int G_R = (EPG * C * NODES + 1) / 2 * 2;    // 16 B aligned (cp.async 16)
  static constexpr int G_RP = G_R + EPG * C * NODES;
  static constexpr int GROUP = G_RP + EPG * NODES;
  static constexpr int GROUP_AL = (GROUP + 1) / 2 * 2;            // keep 16 B alignment
  static constexpr int OFF_TAB = GPB * GROUP_AL;
  static constexpr int TOTAL = OFF_TAB + N * N + 2 * N + GeoLayout<D>::STRIDE;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
};

template <int TG>
__device__ __forceinline__ void group_sync(int gid) {
  if (TG == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(gid + 1), "r"(TG) : "memory");
  }
}

// Face integrand u_hat - F_n(own)/2 on a Cartesian face (operator.py:224-240):
// only the normal velocity v_m and p enter; returns (F_v, F_p) * face scale.
// Every rounding is spelled out (no mul+add left for ptxas to contract or not,
// which it decides per kernel and register budget): all kernels that share
// this function produce the same bits -- the cluster kernel, the stream
// kernels and the slab runs are compared bitwise.
__device__ __forceinline__ void cart_face_flux(double vo, double po, double vx, double px,
                                               double nm, double fs, double ir, double c2r,
                                               double tau, double irt, bool stab, double& fv,
                                               double& fp) {
  const double vn_o = __dmul_rn(nm, vo), vn_x = __dmul_rn(nm, vx);
  double pv = __dmul_rn(__dmul_rn(0.5, ir), px);
  double pp = __dmul_rn(__dmul_rn(0.5, c2r), vn_x);
  if (stab) {
    pv = __fma_rn(__dmul_rn(0.5, irt), __dsub_rn(vn_o, vn_x), pv);
    pp = __fma_rn(__dmul_rn(__dmul_rn(0.5, c2r), tau), __dsub_rn(po, px), pp);
  }
  fv = __dmul_rn(__dmul_rn(pv, nm), fs);
  fp = __dmul_rn(pp, fs);
}

template <int D, int N, int MODE>
__global__ void __launch_bounds__(GroupCfg<D, N>::TPB)
affine_group_kernel(const AffineArgs args) {
  using K = GroupCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, EPG = K::EPG, TG = K::TG;
  constexpr bool READ_RV = (MODE == OUT_LSRK) || (MODE == OUT_ADERB);
  extern __shared__ __align__(16) double smem[];
  double* const tabs = smem + K::OFF_TAB;
  double* const geo = tabs + N * N + 2 * N;
  const int tid = threadIdx.x;
  for (int i = tid; i < N * N + 2 * N; i += K::TPB) tabs[i] = args.tab[i];
  for (int i = tid; i < GLy::STRIDE; i += K::TPB) geo[i] = args.geo[i];

  const int gid = tid / TG, lane = tid - gid * TG;
  double* const su = smem + gid * K::GROUP_AL + K::G_U;
  double* const sr = smem + gid * K::GROUP_AL + K::G_R;
  double* const srp = smem + gid * K::GROUP_AL + K::G_RP;
  const long long e_end = args.e_begin + args.E;
  const long long e0 = args.e_begin + ((long long)blockIdx.x * K::GPB + gid) * EPG;
  const int nel = (int)max(0LL, min((long long)EPG, e_end - e0));
  const bool faces = (args.parts & PART_FACE) != 0;
  const bool cell = (args.parts & PART_CELL) != 0;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || args.a != 0.0);
  const double* __restrict__ gsrc_r = (MODE == OUT_ADERB) ? args.v : args.r;

  // ---- 1. stream the u tile in (cp.async), meanwhile fetch this lane's
  //         neighbour face values (v_m, p at both ends of its d pencils) ----
  if (nel > 0) {
    const int tot = nel * C * NODES;
    const double* gu = args.u + e0 * C * NODES;
    const double* gr = gsrc_r + e0 * C * NODES;
    if (((e0 * C * NODES) & 1) == 0) {
      for (int i = 2 * lane; i < tot; i += 2 * TG) {
        if (i + 1 < tot) {
          cp_async16(su + i, gu + i);
          if (read_r) cp_async16(sr + i, gr + i);
        } else {
          cp_async8(su + i, gu + i);
          if (read_r) cp_async8(sr + i, gr + i);
        }
      }
    } else {
      for (int i = lane; i < tot; i += TG) {
        cp_async8(su + i, gu + i);
        if (read_r) cp_async8(sr + i, gr + i);
      }
    }
  }
  cp_async_commit();
  const int q = lane / NF, fn = lane - (lane / NF) * NF;
  const bool plane = lane < EPG * NF && q < nel;
  const long long e = e0 + q;
  double nbv[D][2][2];   // [m][side][v_m, p] neighbour trace values
  int nbk[D][2];
  double ir = 0.0, c2r = 0.0, tau = 1.0, irt = 0.0;
  if (plane) {
    const double* mt = args.mat + e * kMatStride;
    ir = __ldg(mt + 0);
    c2r = __ldg(mt + 1);
    tau = __ldg(mt + 2);
    irt = __ldg(mt + 3);
    // all neighbour ids first, then every value load unconditionally from a
    // valid address (walls read the own element), so the loads batch
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
      for (int s = 0; s < 2; ++s)
        nbk[m][s] = faces ? __ldg(args.nbr + e * 2 * D + 2 * m + s) : -1;
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int nb = nbk[m][s];
        WK_CHECK_NBR(args, nb);
        const bool ghost = nb <= -2;
        const double* src = ghost ? args.ghost + (long long)ghost_slot(nb) * C * NF + fn
                                  : args.u + (long long)(nb >= 0 ? nb : e) * C * NODES +
                                        face_to_node<N>(m, 1 - s, fn);
        const int cs = ghost ? NF : NODES;
        nbv[m][s][0] = __ldg(src + m * cs);
        nbv[m][s][1] = __ldg(src + D * cs);
      }
  }
  cp_async_wait<0>();
  __syncthreads();  // u tiles and the CTA tables are visible

  // ---- 2. pencils: direction m, face position fn ------------------------
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
    if (plane) {
      const int nb0 = pencil_base<N>(m, fn);   // node with i_m = 0
      const long long gbase = e * C * NODES + nb0;
      const double* rl = sr + q * C * NODES + nb0;
      const double* ul = su + q * C * NODES + nb0;
      double pl[N], vl[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        pl[i] = ul[D * NODES + i * sm];
        vl[i] = ul[m * NODES + i * sm];
      }
      // the two faces this pencil pierces
      double fv0 = 0.0, fp0 = 0.0, fv1 = 0.0, fp1 = 0.0;
      if (faces) {
        const double nm0 = geo[GLy::NORMAL + (m * 2 + 0) * D + m];
        const double nm1 = geo[GLy::NORMAL + (m * 2 + 1) * D + m];
        const double fs0 = geo[GLy::FSCALE + m * 2 + 0];
        const double fs1 = geo[GLy::FSCALE + m * 2 + 1];
        const bool w0 = nbk[m][0] == -1, w1 = nbk[m][1] == -1;  // sound-soft mirror
        cart_face_flux(vl[0], pl[0], w0 ? vl[0] : nbv[m][0][0], w0 ? -pl[0] : nbv[m][0][1],
                       nm0, fs0, ir, c2r, tau, irt, args.stab, fv0, fp0);
        cart_face_flux(vl[N - 1], pl[N - 1], w1 ? vl[N - 1] : nbv[m][1][0],
                       w1 ? -pl[N - 1] : nbv[m][1][1], nm1, fs1, ir, c2r, tau, irt,
                       args.stab, fv1, fp1);
      }
      const double gmm = geo[m * D + m];
      const double cv = cell ? ir * gmm : 0.0;
      const double cp = cell ? c2r * gmm : 0.0;
      double* rpl = srp + q * NODES + nb0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double ap = 0.0, av = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double a = args.cA[i * N + j];   // constant-bank operand
          ap = fma(a, pl[j], ap);
          av = fma(a, vl[j], av);
        }
        const double l0 = args.cL0[i], l1 = args.cL1[i];
        const double resv = fma(cv, ap, fma(l0, fv0, l1 * fv1));
        double resp = fma(cp, av, fma(l0, fp0, l1 * fp1));
        if (m > 0) resp += rpl[i * sm];
        // v_m is final after direction m
        const long long iv = gbase + m * NODES + i * sm;
        if (MODE == OUT_MINVK) {
          args.out[iv] = resv;
        } else if (MODE == OUT_RHS) {
          args.out[iv] = -resv;
        } else if (MODE == OUT_LSRK) {
          const double f = -resv * args.dt;
          const double rr = read_r ? fma(args.a, rl[m * NODES + i * sm], f) : f;
          args.r[iv] = rr;
          args.u_out[iv] = fma(args.b, rr, vl[i]);
        } else if (MODE == OUT_ADERB) {
          args.out[iv] = rl[m * NODES + i * sm] - resv;
        }
        if (m < D - 1) {
          rpl[i * sm] = resp;
        } else {
          const long long ip = gbase + D * NODES + i * sm;
          if (MODE == OUT_MINVK) {
            args.out[ip] = resp;
          } else if (MODE == OUT_RHS) {
            args.out[ip] = -resp;
          } else if (MODE == OUT_LSRK) {
            const double f = -resp * args.dt;
            const double rr = read_r ? fma(args.a, rl[D * NODES + i * sm], f) : f;
            args.r[ip] = rr;
            args.u_out[ip] = fma(args.b, rr, pl[i]);
          } else if (MODE == OUT_ADERB) {
            args.out[ip] = rl[D * NODES + i * sm] - resp;
          }
        }
      }
    }
    if (m < D - 1) group_sync<TG>(gid);
  }
}

}  // namespace wk
