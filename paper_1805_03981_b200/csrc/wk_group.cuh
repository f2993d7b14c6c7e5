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
  static constexpr int NB2 = 2 * D * 2 * NF;                       // staged face values / element
  // per-group smem (doubles): u | nb (v_m, p per face node) | Rp | mat
  static constexpr int G_U = 0;
  static constexpr int G_NB = EPG * C * NODES;
  static constexpr int G_RP = G_NB + EPG * NB2;
  static constexpr int G_MAT = G_RP + EPG * NODES;
  static constexpr int GROUP = G_MAT + EPG * kMatStride;
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
  __syncthreads();  // the only CTA-wide barrier

  const int gid = tid / TG, lane = tid - gid * TG;
  double* const gs = smem + gid * K::GROUP_AL;
  double* const su = gs + K::G_U;
  double* const snb = gs + K::G_NB;
  double* const srp = gs + K::G_RP;
  double* const smt = gs + K::G_MAT;
  const long long e_end = args.e_begin + args.E;
  const long long e0 = args.e_begin + ((long long)blockIdx.x * K::GPB + gid) * EPG;
  if (e0 >= e_end) return;
  const int nel = (int)min((long long)EPG, e_end - e0);
  const bool faces = (args.parts & PART_FACE) != 0;
  const bool cell = (args.parts & PART_CELL) != 0;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || args.a != 0.0);
  const double* __restrict__ gsrc_r = (MODE == OUT_ADERB) ? args.v : args.r;

  // ---- 1. stage u, material and the neighbour (v_m, p) face values ---------
  {
    const int tot = nel * C * NODES;
    const double* gu = args.u + e0 * C * NODES;
    if (((e0 * C * NODES) & 1) == 0) {
      for (int i = 2 * lane; i < tot; i += 2 * TG) {
        if (i + 1 < tot) cp_async16(su + i, gu + i); else cp_async8(su + i, gu + i);
      }
    } else {
      for (int i = lane; i < tot; i += TG) cp_async8(su + i, gu + i);
    }
    for (int i = lane; i < nel * kMatStride; i += TG)
      cp_async8(smt + i, args.mat + e0 * kMatStride + i);
    if (faces) {
#pragma unroll
      for (int f = 0; f < 2 * D; ++f) {
        const int m = f >> 1, sd = f & 1;
        for (int idx = lane; idx < nel * NF; idx += TG) {
          const int q = idx / NF, fn = idx - (idx / NF) * NF;
          const int nb = __ldg(args.nbr + (e0 + q) * 2 * D + f);
          double* dst = snb + (q * 2 * D + f) * 2 * NF + fn;
          if (nb >= 0) {
            const double* src = args.u + (long long)nb * C * NODES +
                                face_to_node<N>(m, 1 - sd, fn);
            cp_async8(dst, src + m * NODES);
            cp_async8(dst + NF, src + D * NODES);
          } else if (nb <= -2) {
            const double* src = args.ghost + (long long)ghost_slot(nb) * C * NF + fn;
            cp_async8(dst, src + m * NF);
            cp_async8(dst + NF, src + D * NF);
          }
        }
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    group_sync<TG>(gid);
  }

  // ---- 2. face integrands (operator.py:224-240), in place -----------------
  if (faces) {
#pragma unroll
    for (int f = 0; f < 2 * D; ++f) {
      const int m = f >> 1, sd = f & 1;
      const double nm = geo[GLy::NORMAL + (m * 2 + sd) * D + m];  // +-1
      const double fs = geo[GLy::FSCALE + m * 2 + sd];
      for (int idx = lane; idx < nel * NF; idx += TG) {
        const int q = idx / NF, fn = idx - (idx / NF) * NF;
        const int nb = __ldg(args.nbr + (e0 + q) * 2 * D + f);
        const double* uq = su + q * C * NODES + face_to_node<N>(m, sd, fn);
        const double vo = uq[m * NODES], po = uq[D * NODES];
        double* slot = snb + (q * 2 * D + f) * 2 * NF + fn;
        double vx, px;
        if (nb == -1) {  // sound-soft mirror
          vx = vo;
          px = -po;
        } else {
          vx = slot[0];
          px = slot[NF];
        }
        const double* mq = smt + q * kMatStride;
        const double ir = mq[0], c2r = mq[1], tau = mq[2], irt = mq[3];
        const double vn_o = nm * vo, vn_x = nm * vx;
        double pv = 0.5 * ir * px;
        double pp = 0.5 * c2r * vn_x;
        if (args.stab) {
          pv += 0.5 * irt * (vn_o - vn_x);
          pp += 0.5 * c2r * tau * (po - px);
        }
        slot[0] = pv * nm * fs;
        slot[NF] = pp * fs;
      }
    }
    group_sync<TG>(gid);
  }

  // ---- 3. pencils, one direction at a time --------------------------------
  const double* sA = tabs;
  const double* sL0 = tabs + N * N;
  const double* sL1 = sL0 + N;
  const int q = lane / NF, fn = lane - (lane / NF) * NF;
  const bool plane = lane < EPG * NF && q < nel;
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
    if (plane) {
      const int nb0 = pencil_base<N>(m, fn);   // node with i_m = 0
      const long long gbase = (e0 + q) * C * NODES + nb0;
      // r / V for the v_m line (and the p line on the last direction)
      double rv[N], rp[N];
      if (read_r) {
#pragma unroll
        for (int i = 0; i < N; ++i) rv[i] = __ldg(gsrc_r + gbase + m * NODES + i * sm);
        if (m == D - 1) {
#pragma unroll
          for (int i = 0; i < N; ++i) rp[i] = __ldg(gsrc_r + gbase + D * NODES + i * sm);
        }
      }
      const double* ul = su + q * C * NODES + nb0;
      double pl[N], vl[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        pl[i] = ul[D * NODES + i * sm];
        vl[i] = ul[m * NODES + i * sm];
      }
      const double gmm = geo[m * D + m];
      const double cv = cell ? smt[q * kMatStride + 0] * gmm : 0.0;
      const double cp = cell ? smt[q * kMatStride + 1] * gmm : 0.0;
      double fv0 = 0.0, fv1 = 0.0, fp0 = 0.0, fp1 = 0.0;
      if (faces) {
        const double* f0 = snb + (q * 2 * D + 2 * m) * 2 * NF + fn;
        fv0 = f0[0];
        fp0 = f0[NF];
        fv1 = f0[2 * NF];
        fp1 = f0[3 * NF];
      }
      double* rpl = srp + q * NODES + nb0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double ap = 0.0, av = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double a = sA[i * N + j];
          ap = fma(a, pl[j], ap);
          av = fma(a, vl[j], av);
        }
        const double l0 = sL0[i], l1 = sL1[i];
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
          const double rr = read_r ? fma(args.a, rv[i], f) : f;
          args.r[iv] = rr;
          args.u_out[iv] = fma(args.b, rr, vl[i]);
        } else if (MODE == OUT_ADERB) {
          args.out[iv] = rv[i] - resv;
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
            const double rr = read_r ? fma(args.a, rp[i], f) : f;
            args.r[ip] = rr;
            args.u_out[ip] = fma(args.b, rr, pl[i]);
          } else if (MODE == OUT_ADERB) {
            args.out[ip] = rp[i] - resp;
          }
        }
      }
    }
    if (m < D - 1) group_sync<TG>(gid);
  }
}

}  // namespace wk
