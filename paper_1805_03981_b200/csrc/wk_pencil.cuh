// Pencil-parallel fused operator for axis-aligned (Cartesian) affine cells —
// the hot path of BASELINE configs 1, 2, 4 and 5.
//
// Same arithmetic as wk_affine.cuh (collapsed split form, see there), mapped
// for shared-memory bandwidth.  On a Cartesian cell G is diagonal and every
// face normal is +-e_m, so
//
//   (M^{-1}K u)_{v_m} = ir G_mm A_m p + L0 (x) F^{v}_{m,0} + L1 (x) F^{v}_{m,1}
//   (M^{-1}K u)_p     = sum_m [ c2r G_mm A_m v_m + L0 (x) F^{p}_{m,0} + L1 (x) F^{p}_{m,1} ]
//
// i.e. v_m is produced entirely by 1-D work along direction m.  One thread
// owns one pencil (a line of n nodes along m): it loads the p- and v_m-lines
// once (n loads for n^2 FMAs, against one load per FMA in a node-per-thread
// mapping), adds its two face lifts and writes the v_m result and its share
// of p.  A node-per-thread epilogue sums the d shares of p and applies the
// LSRK / ADER update with coalesced global stores.
//
// Schedule per tile of EPB elements (persistent CTAs):
//   * u tile t+1 streams global->shared with cp.async while tile t computes;
//   * neighbour face-node values of tile t+1 are prefetched into registers,
//     the register state r / V of tile t+1 likewise;
//   * face integrands (2 non-zero components on Cartesian faces) -> smem,
//     pencils -> smem results, epilogue -> global.
#pragma once
#include "wk_stage.cuh"

namespace wk {

template <int D, int N>
struct PencilCfg {
  static constexpr int C = D + 1;
  static constexpr int NODES = D == 3 ? N * N * N : N * N;
  static constexpr int NF = D == 3 ? N * N : N;
  static constexpr int TPB = 256;
  static constexpr int PENC = D * NF;                    // pencils per element
  static constexpr int EPB = PENC >= TPB ? 1 : TPB / PENC;
  static constexpr int TILE = EPB * C * NODES;
  static constexpr int FSL = EPB * 2 * D * NF;           // face slots per tile
  static constexpr int SPT = (FSL + TPB - 1) / TPB;      // face slots per thread
  static constexpr int NPT = (EPB * NODES + TPB - 1) / TPB;  // epilogue nodes per thread
  static constexpr int PPT = (EPB * PENC + TPB - 1) / TPB;   // pencils per thread
  // smem (doubles): u[2] | mat[2] | F | Rv | Rp | tabs | geo
  static constexpr int MAT = EPB * kMatStride;
  // u stages start on 16-byte boundaries (16-byte cp.async fills them)
  static constexpr int TILE_AL = (TILE + 1) / 2 * 2;
  static constexpr int OFF_U0 = 0;
  static constexpr int OFF_U1 = TILE_AL;
  static constexpr int OFF_M0 = 2 * TILE_AL;
  static constexpr int OFF_M1 = OFF_M0 + MAT;
  static constexpr int OFF_F = OFF_M1 + MAT;
  static constexpr int OFF_RV = OFF_F + EPB * 2 * D * 2 * NF;
  static constexpr int OFF_RP = OFF_RV + EPB * D * NODES;
  static constexpr int OFF_TAB = OFF_RP + EPB * D * NODES;
  static constexpr int OFF_GEO = OFF_TAB + N * N + 2 * N;
  static constexpr int TOTAL = OFF_GEO + GeoLayout<D>::STRIDE;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
};

template <int D, int N, int MODE>
__global__ void __launch_bounds__(256, 2)
affine_pencil_kernel(const AffineArgs args) {
  using K = PencilCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, EPB = K::EPB, TPB = K::TPB;
  constexpr int SPT = K::SPT, NPT = K::NPT, PPT = K::PPT;
  constexpr bool READ_RV = (MODE == OUT_LSRK) || (MODE == OUT_ADERB);
  extern __shared__ __align__(16) double smem[];
  double* const sF = smem + K::OFF_F;
  double* const sRv = smem + K::OFF_RV;
  double* const sRp = smem + K::OFF_RP;
  double* const tabs = smem + K::OFF_TAB;
  double* const geo = smem + K::OFF_GEO;
  const int tid = threadIdx.x;
  const bool faces = (args.parts & PART_FACE) != 0;
  const bool cell = (args.parts & PART_CELL) != 0;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || args.a != 0.0);
  const long long e_end = args.e_begin + args.E;
  const long long ntiles = (args.E + EPB - 1) / EPB;
  const double* __restrict__ gsrc_r = (MODE == OUT_ADERB) ? args.v : args.r;

  for (int i = tid; i < N * N + 2 * N; i += TPB) tabs[i] = args.tab[i];
  for (int i = tid; i < GLy::STRIDE; i += TPB) geo[i] = args.geo[i];

  // ---- fixed per-thread work lists ---------------------------------------
  // face slots: (element, face f, face node fn)
  int f_el[SPT], f_f[SPT], f_fn[SPT], f_own[SPT], f_nbn[SPT];
#pragma unroll
  for (int j = 0; j < SPT; ++j) {
    const int s = tid + j * TPB;
    const int fn = s % NF, rest = s / NF;
    const int f = rest % (2 * D), q = rest / (2 * D);
    f_el[j] = s < K::FSL ? q : EPB;
    f_f[j] = f;
    f_fn[j] = fn;
    f_own[j] = q * C * NODES + face_to_node<N>(f >> 1, f & 1, fn);
    f_nbn[j] = face_to_node<N>(f >> 1, 1 - (f & 1), fn);
  }
  // epilogue nodes
  int n_el[NPT], n_node[NPT];
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int s = tid + j * TPB;
    n_el[j] = s < EPB * NODES ? s / NODES : EPB;
    n_node[j] = s % NODES;
  }

  long long tile = blockIdx.x;
  if (tile >= ntiles) return;

  // registers prefetched one tile ahead: neighbour face values, r / V values
  double nbv[SPT][C];
  int nbk[SPT];          // neighbour code of the prefetched slot (-1 wall)
  double rpre[NPT][C];

  auto prefetch_regs = [&](long long t) {
    const long long e0 = args.e_begin + t * EPB;
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
      const long long e = e0 + f_el[j];
      int nb = -1;
      if (f_el[j] < EPB && e < e_end && faces) nb = __ldg(args.nbr + e * 2 * D + f_f[j]);
      nbk[j] = nb;
      WK_CHECK_NBR(args, nb);
      if (nb >= 0) {
        const double* src = args.u + (long long)nb * C * NODES + f_nbn[j];
#pragma unroll
        for (int c = 0; c < C; ++c) nbv[j][c] = __ldg(src + c * NODES);
      } else if (nb <= -2) {
        const double* src = args.ghost + (long long)ghost_slot(nb) * C * NF + f_fn[j];
#pragma unroll
        for (int c = 0; c < C; ++c) nbv[j][c] = __ldg(src + c * NF);
      }
    }
    if (read_r) {
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const long long e = e0 + n_el[j];
        if (n_el[j] < EPB && e < e_end) {
          const double* src = gsrc_r + e * C * NODES + n_node[j];
#pragma unroll
          for (int c = 0; c < C; ++c) rpre[j][c] = __ldg(src + c * NODES);
        }
      }
    }
  };
  auto issue_u = [&](long long t, double* su, double* sm_) {
    const long long e0 = args.e_begin + t * EPB;
    const int nel = (int)min((long long)EPB, e_end - e0);
    const int tot = nel * C * NODES;
    const double* gu = args.u + e0 * C * NODES;
    if (((e0 * C * NODES) & 1) == 0) {
      for (int i = 2 * tid; i < tot; i += 2 * TPB) {
        if (i + 1 < tot) cp_async16(su + i, gu + i); else cp_async8(su + i, gu + i);
      }
    } else {
      for (int i = tid; i < tot; i += TPB) cp_async8(su + i, gu + i);
    }
    for (int i = tid; i < nel * kMatStride; i += TPB)
      cp_async8(sm_ + i, args.mat + e0 * kMatStride + i);
  };

  issue_u(tile, smem + K::OFF_U0, smem + K::OFF_M0);
  cp_async_commit();
  prefetch_regs(tile);
  int buf = 0;

  for (; tile < ntiles; tile += gridDim.x) {
    const long long nxt = tile + gridDim.x;
    const double* const su = smem + (buf ? K::OFF_U1 : K::OFF_U0);
    const double* const smt = smem + (buf ? K::OFF_M1 : K::OFF_M0);
    if (nxt < ntiles) issue_u(nxt, smem + (buf ? K::OFF_U0 : K::OFF_U1),
                              smem + (buf ? K::OFF_M0 : K::OFF_M1));
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const long long e0 = args.e_begin + tile * EPB;
    const int nel = (int)min((long long)EPB, e_end - e0);

    // ---- face integrands: v_m and p components (operator.py:224-240) ----
    if (faces) {
#pragma unroll
      for (int j = 0; j < SPT; ++j) {
        const int q = f_el[j];
        if (q >= nel) continue;
        const int f = f_f[j], m = f >> 1, sd = f & 1;
        const double ir = smt[q * kMatStride + 0], c2r = smt[q * kMatStride + 1];
        const double tau = smt[q * kMatStride + 2], irt = smt[q * kMatStride + 3];
        const double vo = su[f_own[j] + m * NODES], po = su[f_own[j] + D * NODES];
        double vx, px;
        if (nbk[j] == -1) {  // sound-soft mirror
          vx = vo;
          px = -po;
        } else {
          vx = nbv[j][m];
          px = nbv[j][D];
        }
        const double nm = geo[GLy::NORMAL + (m * 2 + sd) * D + m];  // +-1
        const double vn_o = nm * vo, vn_x = nm * vx;
        double pv = 0.5 * ir * px;
        double pp = 0.5 * c2r * vn_x;
        if (args.stab) {
          pv += 0.5 * irt * (vn_o - vn_x);
          pp += 0.5 * c2r * tau * (po - px);
        }
        const double fs = geo[GLy::FSCALE + m * 2 + sd];
        double* slot = sF + ((q * 2 * D + f) * 2) * NF + f_fn[j];
        slot[0] = pv * nm * fs;
        slot[NF] = pp * fs;
      }
    }
    // keep this tile's r / V, then prefetch the next tile's neighbour faces
    // and r / V into registers (consumed one iteration later)
    double rcur[NPT][C];
#pragma unroll
    for (int j = 0; j < NPT; ++j)
#pragma unroll
      for (int c = 0; c < C; ++c) rcur[j][c] = rpre[j][c];
    if (nxt < ntiles) prefetch_regs(nxt);
    __syncthreads();

    // ---- pencils: thread (element, direction m, face position fn) --------
    const double* sA = tabs;
    const double* sL0 = tabs + N * N;
    const double* sL1 = sL0 + N;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int s = tid + j * TPB;
      if (s >= EPB * K::PENC) break;
      const int q = s / K::PENC, w = s - q * K::PENC;
      const int m = w / NF, fn = w - m * NF;
      if (q >= nel) continue;
      const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
      const int lo = fn % sm, hi = fn / sm;
      const int nb0 = lo + hi * sm * N;
      const double* pl = su + q * C * NODES + D * NODES + nb0;
      const double* vl = su + q * C * NODES + m * NODES + nb0;
      double pv[N], vv[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        pv[i] = cell ? pl[i * sm] : 0.0;
        vv[i] = cell ? vl[i * sm] : 0.0;
      }
      const double gmm = geo[m * D + m];
      const double cv = smt[q * kMatStride + 0] * gmm;
      const double cp = smt[q * kMatStride + 1] * gmm;
      double fv0 = 0.0, fv1 = 0.0, fp0 = 0.0, fp1 = 0.0;
      if (faces) {
        const double* f0 = sF + ((q * 2 * D + 2 * m) * 2) * NF + fn;
        fv0 = f0[0];
        fp0 = f0[NF];
        fv1 = f0[2 * NF];
        fp1 = f0[3 * NF];
      }
      double* rv = sRv + (q * D + m) * NODES + nb0;
      double* rp = sRp + (q * D + m) * NODES + nb0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double ap = 0.0, av = 0.0;
#pragma unroll
        for (int jj = 0; jj < N; ++jj) {
          const double a = sA[i * N + jj];
          ap = fma(a, pv[jj], ap);
          av = fma(a, vv[jj], av);
        }
        const double l0 = sL0[i], l1 = sL1[i];
        rv[i * sm] = fma(cv, ap, fma(l0, fv0, l1 * fv1));
        rp[i * sm] = fma(cp, av, fma(l0, fp0, l1 * fp1));
      }
    }
    __syncthreads();

    // ---- epilogue: node per thread, coalesced stores ----------------------
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int q = n_el[j];
      if (q >= nel) continue;
      const int node = n_node[j];
      double res[C];
      double p = 0.0;
#pragma unroll
      for (int m = 0; m < D; ++m) {
        res[m] = sRv[(q * D + m) * NODES + node];
        p += sRp[(q * D + m) * NODES + node];
      }
      res[D] = p;
      const long long gb = (e0 + q) * C * NODES + node;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const long long idx = gb + c * NODES;
        if (MODE == OUT_MINVK) {
          args.out[idx] = res[c];
        } else if (MODE == OUT_RHS) {
          args.out[idx] = -res[c];
        } else if (MODE == OUT_LSRK) {
          const double f = -res[c] * args.dt;
          const double rr = read_r ? fma(args.a, rcur[j][c], f) : f;
          args.r[idx] = rr;
          args.u_out[idx] = fma(args.b, rr, su[q * C * NODES + c * NODES + node]);
        } else if (MODE == OUT_ADERB) {
          args.out[idx] = rcur[j][c] - res[c];
        }
      }
    }
    __syncthreads();  // u stage, F and R are reused next iteration
    buf ^= 1;
  }
}

}  // namespace wk
