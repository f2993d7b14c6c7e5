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
  // one pipeline stage: u | r-or-v | nb | mat | geo (geo only for multi-class)
  static constexpr int STAGE = 2 * TILE + NBT + MAT + GEO;
  static constexpr int TAB = N * N + 2 * N;
  static constexpr int WS = EPB * D * NODES;            // non-Cartesian flux combos
  static constexpr size_t BYTES = sizeof(double) * (2 * STAGE + TAB + GeoLayout<D>::STRIDE + WS);
};

template <int D, int N, bool CART, int MODE>
__global__ void __launch_bounds__(Shape<D, N>::TPB)
affine_stage_kernel(AffineArgs args) {
  using K = StageCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, EPB = K::EPB, TPB = K::TPB;
  constexpr bool READ_RV = (MODE == OUT_LSRK) || (MODE == OUT_ADERB);
  extern __shared__ __align__(16) double smem[];
  double* stage[2] = {smem, smem + K::STAGE};
  double* tabs = smem + 2 * K::STAGE;
  double* geo0 = tabs + K::TAB;
  double* ws = geo0 + GLy::STRIDE;
  const int tid = threadIdx.x;
  const bool faces = (args.parts & PART_FACE) != 0;
  const bool cell = (args.parts & PART_CELL) != 0;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || args.a != 0.0);
  const bool multi = args.geo_class != nullptr;
  const long long e_end = args.e_begin + args.E;
  const long long ntiles = (args.E + EPB - 1) / EPB;

  for (int i = tid; i < K::TAB; i += TPB) tabs[i] = args.tab[i];
  if (!multi)
    for (int i = tid; i < GLy::STRIDE; i += TPB) geo0[i] = args.geo[i];

  // fixed per-thread face slots: (el, f, fn) and the two node offsets
  int s_el[K::SPT], s_f[K::SPT], s_fn[K::SPT], s_nbnode[K::SPT], s_own[K::SPT];
#pragma unroll
  for (int j = 0; j < K::SPT; ++j) {
    const int slot = tid + j * TPB;
    const int fn = slot % NF, rest = slot / NF;
    const int f = rest % (2 * D), el = rest / (2 * D);
    s_el[j] = slot < K::SLOTS ? el : -1;
    s_f[j] = f;
    s_fn[j] = fn;
    const int m = f >> 1, sd = f & 1;
    s_nbnode[j] = face_to_node<N>(m, 1 - sd, fn);
    s_own[j] = face_to_node<N>(m, sd, fn);
  }
  const int el = tid / NODES;
  const int node = tid - el * NODES;
  const bool vthread = el < EPB;
  int im[D];
#pragma unroll
  for (int m = 0; m < D; ++m) im[m] = (node / ipow<N>(m)) % N;

  // neighbour ids (per face slot) of the tile after next
  int nbr_next[K::SPT];
  auto fetch_nbr = [&](long long tile, int (&dst)[K::SPT]) {
#pragma unroll
    for (int j = 0; j < K::SPT; ++j) {
      dst[j] = -1;
      if (s_el[j] < 0) continue;
      const long long e = args.e_begin + tile * EPB + s_el[j];
      if (tile < ntiles && e < e_end) dst[j] = __ldg(args.nbr + e * 2 * D + s_f[j]);
    }
  };
  auto issue = [&](long long tile, double* st, const int (&nbr)[K::SPT]) {
    const long long e0 = args.e_begin + tile * EPB;
    const int nel = (int)((e_end - e0) < EPB ? (e_end - e0) : EPB);
    const int tot = nel * C * NODES;
    double* su = st;
    double* sr = st + K::TILE;
    if (((e0 * C * NODES) & 1) == 0) {  // 16-byte aligned tile start
      const double* gu = args.u + e0 * C * NODES;
      for (int i = 2 * tid; i < tot; i += 2 * TPB) {
        if (i + 1 < tot) cp_async16(su + i, gu + i);
        else cp_async8(su + i, gu + i);
      }
      if (read_r) {
        const double* gr = (MODE == OUT_ADERB ? args.v : args.r) + e0 * C * NODES;
        for (int i = 2 * tid; i < tot; i += 2 * TPB) {
          if (i + 1 < tot) cp_async16(sr + i, gr + i);
          else cp_async8(sr + i, gr + i);
        }
      }
    } else {
      const double* gu = args.u + e0 * C * NODES;
      for (int i = tid; i < tot; i += TPB) cp_async8(su + i, gu + i);
      if (read_r) {
        const double* gr = (MODE == OUT_ADERB ? args.v : args.r) + e0 * C * NODES;
        for (int i = tid; i < tot; i += TPB) cp_async8(sr + i, gr + i);
      }
    }
    double* snb = st + 2 * K::TILE;
    if (faces) {
#pragma unroll
      for (int j = 0; j < K::SPT; ++j) {
        const int nb = nbr[j];
        if (s_el[j] < 0 || s_el[j] >= nel || nb == -1) continue;
        double* dst = snb + ((s_el[j] * 2 * D + s_f[j]) * C) * NF + s_fn[j];
        if (nb >= 0) {
          const double* src = args.u + (long long)nb * C * NODES + s_nbnode[j];
#pragma unroll
          for (int c = 0; c < C; ++c) cp_async8(dst + c * NF, src + c * NODES);
        } else {
          const double* src = args.ghost + (long long)ghost_slot(nb) * C * NF + s_fn[j];
#pragma unroll
          for (int c = 0; c < C; ++c) cp_async8(dst + c * NF, src + c * NF);
        }
      }
    }
    double* smt = st + 2 * K::TILE + K::NBT;
    for (int i = tid; i < nel * kMatStride; i += TPB) cp_async8(smt + i, args.mat + e0 * kMatStride + i);
    if (multi) {
      double* sg = smt + K::MAT;
      for (int i = tid; i < nel * GLy::STRIDE; i += TPB) {
        const int q = i / GLy::STRIDE, w = i - q * GLy::STRIDE;
        const int cls = __ldg(args.geo_class + e0 + q);
        cp_async8(sg + i, args.geo + (long long)cls * GLy::STRIDE + w);
      }
    }
  };

  long long tile = blockIdx.x;
  if (tile >= ntiles) return;
  int nbr_cur[K::SPT], nbr_nn[K::SPT];
  fetch_nbr(tile, nbr_cur);
  issue(tile, stage[0], nbr_cur);
  cp_async_commit();
  fetch_nbr(tile + gridDim.x, nbr_next);
  int buf = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    const long long nxt = tile + gridDim.x;
    if (nxt < ntiles) issue(nxt, stage[buf ^ 1], nbr_next);
    cp_async_commit();
    fetch_nbr(nxt + gridDim.x, nbr_nn);
    cp_async_wait<1>();
    __syncthreads();

    double* st = stage[buf];
    double* su = st;
    double* sr = st + K::TILE;
    double* snb = st + 2 * K::TILE;
    double* smt = st + 2 * K::TILE + K::NBT;
    double* sgeo = smt + K::MAT;
    const long long e0 = args.e_begin + tile * EPB;
    const int nel = (int)((e_end - e0) < EPB ? (e_end - e0) : EPB);

    // face integrands, in place over the neighbour slices (operator.py:224-240)
    if (faces) {
#pragma unroll
      for (int j = 0; j < K::SPT; ++j) {
        const int q = s_el[j];
        if (q < 0 || q >= nel) continue;
        const int f = s_f[j], m = f >> 1, sd = f & 1;
        const double* g = multi ? sgeo + q * GLy::STRIDE : geo0;
        const double ir = smt[q * kMatStride + 0], c2r = smt[q * kMatStride + 1];
        const double tau = smt[q * kMatStride + 2];
        double own[C], oth[C];
        double* slot = snb + ((q * 2 * D + f) * C) * NF + s_fn[j];
#pragma unroll
        for (int c = 0; c < C; ++c) own[c] = su[(q * C + c) * NODES + s_own[j]];
        if (nbr_cur[j] == -1) {
#pragma unroll
          for (int c = 0; c < D; ++c) oth[c] = own[c];
          oth[D] = -own[D];
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) oth[c] = slot[c * NF];
        }
        double nrm[D], vn_o = 0.0, vn_x = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          nrm[i] = g[GLy::NORMAL + (m * 2 + sd) * D + i];
          vn_o = fma(nrm[i], own[i], vn_o);
          vn_x = fma(nrm[i], oth[i], vn_x);
        }
        double pv = 0.5 * ir * oth[D];
        double pp = 0.5 * c2r * vn_x;
        if (args.stab) {
          pv += 0.5 * ir / tau * (vn_o - vn_x);
          pp += 0.5 * c2r * tau * (own[D] - oth[D]);
        }
        const double fs = g[GLy::FSCALE + m * 2 + sd];
#pragma unroll
        for (int i = 0; i < D; ++i) slot[i * NF] = pv * nrm[i] * fs;
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
        for (int i = 0; i < D; ++i) w = fma(g[m * D + i], su[(el * C + i) * NODES + node], w);
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
        const double* up = su + (el * C + D) * NODES;
#pragma unroll
        for (int m = 0; m < D; ++m) {
          const int sm = ipow<N>(m);
          const int base = node - im[m] * sm;
          const double* arow = sA + im[m] * N;
          const double* wl = CART ? su + (el * C + m) * NODES : ws + (el * D + m) * NODES;
          double dp = 0.0, dw = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const double a = arow[j];
            dp = fma(a, up[base + j * sm], dp);
            dw = fma(a, wl[base + j * sm], dw);
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
      const long long base = (e0 + el) * C * NODES + node;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const long long idx = base + c * NODES;
        const double uv = su[(el * C + c) * NODES + node];
        if (MODE == OUT_MINVK) {
          args.out[idx] = res[c];
        } else if (MODE == OUT_RHS) {
          args.out[idx] = -res[c];
        } else if (MODE == OUT_LSRK) {
          const double f = -res[c] * args.dt;
          const double rr = read_r ? fma(args.a, sr[(el * C + c) * NODES + node], f) : f;
          args.r[idx] = rr;
          args.u_out[idx] = fma(args.b, rr, uv);
        } else if (MODE == OUT_ADERB) {
          args.out[idx] = sr[(el * C + c) * NODES + node] - res[c];
        }
      }
    }
    __syncthreads();  // stage[buf] is refilled by the next iteration's issue
#pragma unroll
    for (int j = 0; j < K::SPT; ++j) {
      nbr_cur[j] = nbr_next[j];
      nbr_next[j] = nbr_nn[j];
    }
    buf ^= 1;
  }
}

}  // namespace wk
