// Persistent, cp.async-pipelined affine operator kernel (LSRK stage, rhs,
// M^{-1}K, ADER final combination).  Same arithmetic as affine_op_kernel
// (wk_affine.cuh, see the formulation there); different schedule:
//
//  * grid = k x #SMs CTAs that loop over tiles of EPB consecutive elements;
//  * tile t+1's own state (u, and r / V when the mode reads them) and its 2d
//    neighbour face-node slices are copied global->shared with cp.async
//    (LDGSTS) into the second stage buffer while tile t is computed; the
//    neighbour ids of tile t+2 are fetched one iteration earlier still;
//  * every thread owns a fixed list of face-node slots and one volume node,
//    so all index arithmetic is hoisted out of the tile loop;
//  * geometry of single-class meshes (all uniform Cartesian configs) is read
//    into shared memory once per CTA.
#pragma once
#include "wk_affine.cuh"

namespace wk {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND));
}

template <int D, int N>
struct StageCfg {
  using S = Shape<D, N>;
  static constexpr int C = S::C, NODES = S::NODES, NF = S::NF, EPB = S::EPB, TPB = S::TPB;
  static constexpr int TILE = EPB * C * NODES;          // doubles of u (or r) per tile
  static constexpr int NBT = EPB * 2 * D * C * NF;      // doubles of face slices per tile
  static constexpr int SLOTS = EPB * 2 * D * NF;        // face-node slots per tile
  static constexpr int SPT = (SLOTS + TPB - 1) / TPB;   // slots per thread
  static constexpr int MAT = EPB * kMatStride;
  static constexpr int GEO = EPB * GeoLayout<D>::STRIDE;
  // one pipeline stage: u | r-or-v | nb | mat | geo (geo only for multi-class).
  // Every piece starts on a 16-byte boundary: the u and r tiles are filled
  // with 16-byte cp.async, and with an odd tile (odd n in 2-D) or an odd
  // geometry record (2-D: 17 doubles) times an odd EPB the second stage and
  // the r tile used to start 8 bytes off -- a misaligned-address fault once a
  // CTA reached its second tile (2-D k = 5 on 64^2 elements; the "fault above
  // ~2k elements" of round 1).
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  static constexpr int OFF_R = ev(TILE);
  static constexpr int OFF_NB = OFF_R + ev(TILE);
  static constexpr int OFF_MAT = OFF_NB + ev(NBT);
  static constexpr int OFF_GEO = OFF_MAT + ev(MAT);
  static constexpr int STAGE = OFF_GEO + ev(GEO);
  static constexpr int TAB = N * N + 2 * N;
  static constexpr int WS = EPB * D * NODES;            // non-Cartesian flux combos
  static constexpr size_t BYTES = sizeof(double) * (2 * STAGE + TAB + GeoLayout<D>::STRIDE + WS);
};

template <int D, int N>
struct StageMinBlocks {
  static constexpr int v = Shape<D, N>::TPB <= 256 ? 3 : 1;
};

template <int D, int N, bool CART, int MODE>
__global__ void __launch_bounds__(Shape<D, N>::TPB, StageMinBlocks<D, N>::v)
affine_stage_kernel(const AffineArgs args) {
  using K = StageCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, EPB = K::EPB, TPB = K::TPB;
  constexpr int SPT = K::SPT;
  constexpr bool READ_RV = (MODE == OUT_LSRK) || (MODE == OUT_ADERB);
  extern __shared__ __align__(16) double smem[];
  double* const tabs = smem + 2 * K::STAGE;
  double* const geo0 = tabs + K::TAB;
  double* const ws = geo0 + GLy::STRIDE;
  const int tid = threadIdx.x;
  WK_CHECK_SMEM(K::BYTES);
  const bool faces = (args.parts & PART_FACE) != 0;
  const bool cell = (args.parts & PART_CELL) != 0;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || args.a != 0.0);
  const bool multi = args.geo_class != nullptr;
  const long long e_end = args.e_begin + args.E;
  const long long ntiles = (args.E + EPB - 1) / EPB;
  const double* __restrict__ gsrc_r = (MODE == OUT_ADERB) ? args.v : args.r;

  for (int i = tid; i < K::TAB; i += TPB) tabs[i] = args.tab[i];
  if (!multi)
    for (int i = tid; i < GLy::STRIDE; i += TPB) geo0[i] = args.geo[i];

  // fixed per-thread face slots, packed: element-in-tile, face, smem offset
  // of the slot, own-node offset, neighbour-node offset
  int s_el[SPT], s_f[SPT], s_off[SPT], s_own[SPT], s_nbn[SPT];
#pragma unroll
  for (int j = 0; j < SPT; ++j) {
    const int slot = tid + j * TPB;
    const int fn = slot % NF, rest = slot / NF;
    const int f = rest % (2 * D), q = rest / (2 * D);
    s_el[j] = slot < K::SLOTS ? q : EPB;  // EPB = inactive
    s_f[j] = f;
    s_off[j] = ((q * 2 * D + f) * C) * NF + fn;
    s_own[j] = q * C * NODES + face_to_node<N>(f >> 1, f & 1, fn);
    s_nbn[j] = face_to_node<N>(f >> 1, 1 - (f & 1), fn);
  }
  const int el = tid / NODES;
  const int node = tid - el * NODES;
  const bool vthread = el < EPB;
  const int voff = el * C * NODES + node;   // this thread's node, component 0
  int im[D];
#pragma unroll
  for (int m = 0; m < D; ++m) im[m] = (node / ipow<N>(m)) % N;

  long long tile = blockIdx.x;
  if (tile >= ntiles) return;

  int nbr_cur[SPT], nbr_nxt[SPT];
  // prologue: neighbour ids of the first tile, issue its copies
#pragma unroll
  for (int j = 0; j < SPT; ++j) {
    const long long e = args.e_begin + tile * EPB + s_el[j];
    nbr_cur[j] = (s_el[j] < EPB && e < e_end) ? __ldg(args.nbr + e * 2 * D + s_f[j]) : -1;
  }
  int buf = 0;
  // issue tile `tile` into stage 0
  {
    const long long e0 = args.e_begin + tile * EPB;
    const int nel = (int)min((long long)EPB, e_end - e0);
    double* st = smem;
    const int tot = nel * C * NODES;
    const double* gu = args.u + e0 * C * NODES;
    const bool a16 = ((e0 * C * NODES) & 1) == 0;
    for (int i = a16 ? 2 * tid : tid; i < tot; i += a16 ? 2 * TPB : TPB) {
      if (a16 && i + 1 < tot) cp_async16(st + i, gu + i); else cp_async8(st + i, gu + i);
    }
    if (read_r) {
      const double* gr = gsrc_r + e0 * C * NODES;
      for (int i = a16 ? 2 * tid : tid; i < tot; i += a16 ? 2 * TPB : TPB) {
        if (a16 && i + 1 < tot) cp_async16(st + K::OFF_R + i, gr + i);
        else cp_async8(st + K::OFF_R + i, gr + i);
      }
    }
    if (faces) {
#pragma unroll
      for (int j = 0; j < SPT; ++j) {
        const int nb = nbr_cur[j];
        if (s_el[j] >= nel || nb == -1) continue;
        WK_CHECK_NBR(args, nb);
        double* dst = st + K::OFF_NB + s_off[j];
        const double* src = nb >= 0 ? args.u + (long long)nb * C * NODES + s_nbn[j]
                                    : args.ghost + (long long)ghost_slot(nb) * C * NF +
                                          (s_off[j] % NF);
        const int cs = nb >= 0 ? NODES : NF;
#pragma unroll
        for (int c = 0; c < C; ++c) cp_async8(dst + c * NF, src + c * cs);
      }
    }
    for (int i = tid; i < nel * kMatStride; i += TPB)
      cp_async8(st + K::OFF_MAT + i, args.mat + e0 * kMatStride + i);
    if (multi) {
      double* sg = st + K::OFF_GEO;
      for (int i = tid; i < nel * GLy::STRIDE; i += TPB) {
        const int q = i / GLy::STRIDE, w = i - q * GLy::STRIDE;
        const int cls = __ldg(args.geo_class + e0 + q);
        cp_async8(sg + i, args.geo + (long long)cls * GLy::STRIDE + w);
      }
    }
    cp_async_commit();
  }
  // neighbour ids of the second tile
#pragma unroll
  for (int j = 0; j < SPT; ++j) {
    const long long e = args.e_begin + (tile + gridDim.x) * EPB + s_el[j];
    nbr_nxt[j] = (s_el[j] < EPB && e < e_end) ? __ldg(args.nbr + e * 2 * D + s_f[j]) : -1;
  }

  for (; tile < ntiles; tile += gridDim.x) {
    const long long nxt = tile + gridDim.x;
    double* const st = smem + buf * K::STAGE;
    double* const sn = smem + (buf ^ 1) * K::STAGE;
    if (nxt < ntiles) {
      const long long e0 = args.e_begin + nxt * EPB;
      const int nel = (int)min((long long)EPB, e_end - e0);
      const int tot = nel * C * NODES;
      const double* gu = args.u + e0 * C * NODES;
      const bool a16 = ((e0 * C * NODES) & 1) == 0;
      for (int i = a16 ? 2 * tid : tid; i < tot; i += a16 ? 2 * TPB : TPB) {
        if (a16 && i + 1 < tot) cp_async16(sn + i, gu + i); else cp_async8(sn + i, gu + i);
      }
      if (read_r) {
        const double* gr = gsrc_r + e0 * C * NODES;
        for (int i = a16 ? 2 * tid : tid; i < tot; i += a16 ? 2 * TPB : TPB) {
          if (a16 && i + 1 < tot) cp_async16(sn + K::OFF_R + i, gr + i);
          else cp_async8(sn + K::OFF_R + i, gr + i);
        }
      }
      if (faces) {
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
          const int nb = nbr_nxt[j];
          if (s_el[j] >= nel || nb == -1) continue;
          WK_CHECK_NBR(args, nb);
          double* dst = sn + K::OFF_NB + s_off[j];
          const double* src = nb >= 0 ? args.u + (long long)nb * C * NODES + s_nbn[j]
                                      : args.ghost + (long long)ghost_slot(nb) * C * NF +
                                            (s_off[j] % NF);
          const int cs = nb >= 0 ? NODES : NF;
#pragma unroll
          for (int c = 0; c < C; ++c) cp_async8(dst + c * NF, src + c * cs);
        }
      }
      for (int i = tid; i < nel * kMatStride; i += TPB)
        cp_async8(sn + K::OFF_MAT + i, args.mat + e0 * kMatStride + i);
      if (multi) {
        double* sg = sn + K::OFF_GEO;
        for (int i = tid; i < nel * GLy::STRIDE; i += TPB) {
          const int q = i / GLy::STRIDE, w = i - q * GLy::STRIDE;
          const int cls = __ldg(args.geo_class + e0 + q);
          cp_async8(sg + i, args.geo + (long long)cls * GLy::STRIDE + w);
        }
      }
    }
    cp_async_commit();
    // neighbour ids two tiles ahead (latency hidden behind this tile)
    int nbr_nn[SPT];
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
      const long long e = args.e_begin + (nxt + gridDim.x) * EPB + s_el[j];
      nbr_nn[j] = (s_el[j] < EPB && nxt + gridDim.x < ntiles && e < e_end)
                      ? __ldg(args.nbr + e * 2 * D + s_f[j]) : -1;
    }
    cp_async_wait<1>();
    __syncthreads();

    const double* const su = st;
    const double* const sr = st + K::OFF_R;
    double* const snb = st + K::OFF_NB;
    const double* const smt = st + K::OFF_MAT;
    const double* const sgeo = st + K::OFF_GEO;
    const long long e0 = args.e_begin + tile * EPB;
    const int nel = (int)min((long long)EPB, e_end - e0);

    // face integrands, in place over the neighbour slices (operator.py:224-240)
    if (faces) {
#pragma unroll
      for (int j = 0; j < SPT; ++j) {
        const int q = s_el[j];
        if (q >= nel) continue;
        const int f = s_f[j], m = f >> 1, sd = f & 1;
        const double* g = multi ? sgeo + q * GLy::STRIDE : geo0;
        const double ir = smt[q * kMatStride + 0], c2r = smt[q * kMatStride + 1];
        const double tau = smt[q * kMatStride + 2], irt = smt[q * kMatStride + 3];
        double own[C], oth[C];
        double* slot = snb + s_off[j];
#pragma unroll
        for (int c = 0; c < C; ++c) own[c] = su[s_own[j] + c * NODES];
        if (nbr_cur[j] == -1) {
#pragma unroll
          for (int c = 0; c < D; ++c) oth[c] = own[c];
          oth[D] = -own[D];
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) oth[c] = slot[c * NF];
        }
        const double* nr = g + GLy::NORMAL + (m * 2 + sd) * D;
        double nrm[D], vn_o = 0.0, vn_x = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          nrm[i] = nr[i];
          vn_o = fma(nrm[i], own[i], vn_o);
          vn_x = fma(nrm[i], oth[i], vn_x);
        }
        const double fs = g[GLy::FSCALE + m * 2 + sd];
        double pv = 0.5 * ir * oth[D];
        double pp = 0.5 * c2r * vn_x;
        if (args.stab) {
          pv += 0.5 * irt * (vn_o - vn_x);
          pp += 0.5 * c2r * tau * (own[D] - oth[D]);
        }
        pv *= fs;
#pragma unroll
        for (int i = 0; i < D; ++i) slot[i * NF] = pv * nrm[i];
        slot[D * NF] = pp * fs;
      }
    }
    const bool active = vthread && el < nel;
    if (!CART && cell && active) {
      const double* g = multi ? sgeo + el * GLy::STRIDE : geo0;
#pragma unroll
      for (int m = 0; m < D; ++m) {
        double w = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) w = fma(g[m * D + i], su[voff + i * NODES], w);
        ws[(el * D + m) * NODES + node] = w;
      }
    }
    __syncthreads();
    if (active) {
      const double* g = multi ? sgeo + el * GLy::STRIDE : geo0;
      const double* sA = tabs;
      const double* sL0 = tabs + N * N;
      const double* sL1 = sL0 + N;
      double res[C];
#pragma unroll
      for (int c = 0; c < C; ++c) res[c] = 0.0;
      if (cell) {
        const double ir = smt[el * kMatStride + 0], c2r = smt[el * kMatStride + 1];
#pragma unroll
        for (int m = 0; m < D; ++m) {
          const int sm = ipow<N>(m);
          const int lb = voff - im[m] * sm;            // line base, component 0
          const double* arow = sA + im[m] * N;
          const double* pl = su + lb + D * NODES;
          const double* wl = CART ? su + lb + m * NODES : ws + (el * D + m) * NODES + node -
                                                              im[m] * sm;
          double dp = 0.0, dw = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const double a = arow[j];
            dp = fma(a, pl[j * sm], dp);
            dw = fma(a, wl[j * sm], dw);
          }
          if (CART) {
            const double gmm = g[m * D + m];
            res[m] = fma(ir * gmm, dp, res[m]);
            res[D] = fma(c2r * gmm, dw, res[D]);
          } else {
#pragma unroll
            for (int i = 0; i < D; ++i) res[i] = fma(ir * g[m * D + i], dp, res[i]);
            res[D] = fma(c2r, dw, res[D]);
          }
        }
      }
      if (faces) {
#pragma unroll
        for (int m = 0; m < D; ++m) {
          const int sm = ipow<N>(m);
          const int fn = node % sm + (node / (sm * N)) * sm;
          const double l0 = sL0[im[m]], l1 = sL1[im[m]];
          const double* f0 = snb + ((el * 2 * D + 2 * m) * C) * NF + fn;
          const double* f1 = f0 + C * NF;
#pragma unroll
          for (int c = 0; c < C; ++c) res[c] = fma(l0, f0[c * NF], fma(l1, f1[c * NF], res[c]));
        }
      }
      const long long gbase = e0 * C * NODES + voff;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const long long idx = gbase + c * NODES;
        if (MODE == OUT_MINVK) {
          args.out[idx] = res[c];
        } else if (MODE == OUT_RHS) {
          args.out[idx] = -res[c];
        } else if (MODE == OUT_LSRK) {
          const double f = -res[c] * args.dt;
          const double rr = read_r ? fma(args.a, sr[voff + c * NODES], f) : f;
          args.r[idx] = rr;
          args.u_out[idx] = fma(args.b, rr, su[voff + c * NODES]);
        } else if (MODE == OUT_ADERB) {
          args.out[idx] = sr[voff + c * NODES] - res[c];
        }
      }
    }
    __syncthreads();  // stage[buf] is refilled by the next iteration's copies
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
      nbr_cur[j] = nbr_nxt[j];
      nbr_nxt[j] = nbr_nn[j];
    }
    buf ^= 1;
  }
}

}  // namespace wk
