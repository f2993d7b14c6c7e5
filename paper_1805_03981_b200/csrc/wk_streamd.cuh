// Direction-parallel version of the persistent Cartesian stream kernel
// (wk_stream.cuh): the LSRK stage / rhs / M^{-1}K / ADER-B hot path.
//
// affine_stream_kernel gives one element tile to ONE thread group, which
// walks the d directions one after the other: at n = 5 that is a single
// warp per CTA and nine warps per SM, each a serial chain of ~1100
// instructions per tile -- ncu shows the kernel latency-bound (issue slots
// 34 % busy, DRAM 70 %).  Here a CTA is d groups and group m owns direction
// m of the SAME tile: it gathers the two faces its pencils pierce, finishes
// v_m (which only direction m touches on a Cartesian cell) in place and
// leaves its share of p in a partial tile; after one CTA barrier every
// thread sums the d shares for a contiguous slice of nodes and applies the
// update, and after a second barrier one thread sends the tile off with the
// bulk stores.  Same shared memory per CTA (plus two partial tiles), d times
// the warps per SM, a third of the dependent chain per tile.
//
// Arithmetic (expressions and their order) is that of affine_stream_kernel:
// p = (P_0 + P_1) + P_2 equals its running sum bit for bit, so the two
// kernels, and the cluster kernel of wk_small.cuh, give identical results.
//
// Requires whole TMA-aligned tiles (C * NODES even); the launcher falls back
// to affine_stream_kernel otherwise.
#pragma once
#include <type_traits>

#include "wk_stream.cuh"

namespace wk {

template <int D, int N>
struct StreamDCfg {
  using G = GroupCfg<D, N>;
  static constexpr int C = D + 1, NODES = G::NODES, NF = G::NF, EPG = G::EPG, TG = G::TG;
  static constexpr int TPB = D * TG;
  static constexpr int TILE = EPG * C * NODES;
  static constexpr int NBF = EPG * D * 2 * 2 * NF;       // [q][m][side][v_m,p][fn]
  static constexpr int OFF_MAT = (2 * TILE + NBF + 1) / 2 * 2;   // material records (TMA)
  static constexpr int BUF = OFF_MAT + EPG * kMatStride; // one stage: u | r | faces | material
  static constexpr int OFF_P = 2 * BUF;                  // d partial-p tiles
  static constexpr int OFF_BAR = (OFF_P + D * EPG * NODES + 1) / 2 * 2;
  static constexpr int OFF_Q = OFF_BAR + 2;              // two 8-byte mbarriers
  static constexpr int OFF_GEO = OFF_Q + 1;              // two 4-byte tile-queue slots
  static constexpr int TOTAL = OFF_GEO + GeoLayout<D>::STRIDE;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  static constexpr bool ALIGNED = ((C * NODES) % 2) == 0;   // every tile start 16-byte aligned
  // resident CTAs per SM the register allocation is held to: what shared
  // memory allows, as long as 72 registers per thread remain (3-D n = 5: 9
  // CTAs = 27 warps at 72 registers, no spills)
  static constexpr int SMEM_FIT = (int)((227 * 1024) / (BYTES + 1024));
  static constexpr int REG_FIT = 65536 / (TPB * 72);
#ifdef WK_STREAMD_MINB
  static constexpr int MINB = WK_STREAMD_MINB;
#else
  static constexpr int MINB = SMEM_FIT < REG_FIT ? SMEM_FIT : (REG_FIT < 1 ? 1 : REG_FIT);
#endif
};

template <int TPB>
__device__ __forceinline__ void cta_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(TPB) : "memory");
}

// The persistent loop of direction group M.  Tiles are named by their first
// element (32-bit; the launcher checks the range), kNoTile = none.
// FAST: both operator parts with stabilization (every stepper launch) as
// compile-time facts; the stage index of the loop body is a compile-time
// constant as well (the loop is unrolled by two).
template <int D, int N, int MODE, bool FAST, int M>
__device__ __forceinline__ void streamd_run(const AffineArgs& args, double* smem) {
  using K = StreamDCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, EPG = K::EPG, TG = K::TG, TPB = K::TPB;
  constexpr bool READ_RV = (MODE == OUT_LSRK) || (MODE == OUT_ADERB);
  constexpr int sm = M == 0 ? 1 : (M == 1 ? N : N * N);
  constexpr unsigned kNoTile = 0xFFFFFFFFu;
  double* const sP = smem + K::OFF_P;
  unsigned long long* const bar = reinterpret_cast<unsigned long long*>(smem + K::OFF_BAR);
  const double* const geo = smem + K::OFF_GEO;
  const int tid = threadIdx.x;
  const int lane = tid - M * TG;
  const bool leader = (M == 0) && lane == 0;
#ifndef WK_L2_HINT
#define WK_L2_HINT 1
#endif
  const unsigned long long pol = (WK_L2_HINT && leader) ? l2_evict_first_policy() : 0ull;

  const bool faces = FAST || (args.parts & PART_FACE) != 0;
  const bool cell = FAST || (args.parts & PART_CELL) != 0;
  const bool stab = FAST || args.stab != 0;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || args.a != 0.0);
  const double* __restrict__ gsrc_r = (MODE == OUT_ADERB) ? args.v : args.r;
  const unsigned e_end = (unsigned)(args.e_begin + args.E);
  const unsigned ntiles = (unsigned)((args.E + EPG - 1) / EPG);
  // lanes past the last pencil sit the sweeps out (WK_STREAMD_CLAMP=1 lets
  // them repeat the last pencil instead -- no divergent region, but 28 % more
  // FP64 lane work at n = 5: config 5 14.95 -> 15.11 ms/step sustained, and
  // the governor holds the SM clock 50 MHz lower)
#ifndef WK_STREAMD_CLAMP
#define WK_STREAMD_CLAMP 0
#endif
  const int pln = WK_STREAMD_CLAMP ? min(lane, EPG * NF - 1) : lane;
  const bool plane_lane = WK_STREAMD_CLAMP || lane < EPG * NF;
  const int q = pln / NF, fn = pln - (pln / NF) * NF;
  const int nb0 = pencil_base<N>(M, fn);
  // the neighbour's face node opposite this pencil's end s
  const int noff0 = face_to_node<N>(M, 1, fn), noff1 = face_to_node<N>(M, 0, fn);
  const unsigned nb_u32 = smem_u32(smem + 2 * K::TILE + ((q * D + M) * 2 * 2) * NF + fn);

  auto first_elem = [&](unsigned t) -> unsigned {
    return t < ntiles ? (unsigned)tile_elem<EPG>(args, (long long)t) : kNoTile;
  };
  auto fetch_ids = [&](unsigned et, int (&ids)[2]) {
    const unsigned e = et + q;
    const bool ok = faces && plane_lane && et != kNoTile && e < e_end;
    ids[0] = ok ? __ldg(args.nbr + (size_t)e * (2 * D) + 2 * M) : -1;
    ids[1] = ok ? __ldg(args.nbr + (size_t)e * (2 * D) + 2 * M + 1) : -1;
  };
  auto issue = [&](unsigned e0, int b, const int (&ids)[2]) {
    const int nel = (int)min((unsigned)EPG, e_end - e0);
    if (leader) {
      double* su = smem + b * K::BUF;
      const unsigned bytes = (unsigned)(nel * C * NODES * 8);
      const unsigned mbytes = (unsigned)(nel * kMatStride * 8);
      bulk_wait_read<0>();   // the bulk stores that left from this stage have read it
      fence_proxy_async();
      mbar_arrive_expect_tx(&bar[b], (read_r ? 2 * bytes : bytes) + mbytes);
      bulk_g2s(su, args.u + (size_t)e0 * (C * NODES), bytes, &bar[b]);
      if (read_r) {
        if (WK_L2_HINT)
          bulk_g2s_hint(su + K::TILE, gsrc_r + (size_t)e0 * (C * NODES), bytes, &bar[b], pol);
        else
          bulk_g2s(su + K::TILE, gsrc_r + (size_t)e0 * (C * NODES), bytes, &bar[b]);
      }
      bulk_g2s(su + K::OFF_MAT, args.mat + (size_t)e0 * kMatStride, mbytes, &bar[b]);
    }
    if (faces && plane_lane && q < nel) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int nb = ids[s];
        WK_CHECK_NBR(args, nb);
        const unsigned d0 = nb_u32 + (unsigned)(b * K::BUF + s * 2 * NF) * 8u;
        if (nb >= 0) {
          const double* src = args.u + (size_t)nb * (C * NODES) + (s == 0 ? noff0 : noff1);
          cp_async8_u32(d0, src + M * NODES);
          cp_async8_u32(d0 + NF * 8u, src + D * NODES);
        } else if (args.has_ghost && nb <= -2) {
          const double* src = args.ghost + (size_t)ghost_slot(nb) * (C * NF) + fn;
          cp_async8_u32(d0, src + M * NF);
          cp_async8_u32(d0 + NF * 8u, src + D * NF);
        }
      }
    }
  };

  int ids_cur[2], ids_nxt[2], ids_nn[2];
  unsigned e_tile = first_elem(blockIdx.x);
  fetch_ids(e_tile, ids_cur);
  issue(e_tile, 0, ids_cur);
  cp_async_commit();
  // tile queue as in affine_stream_kernel: two static tiles, then claims
  // from the global counter two iterations ahead, published through qslot
  unsigned* const qslot = reinterpret_cast<unsigned*>(smem + K::OFF_Q);
  const unsigned dyn0 = 2u * gridDim.x;
  const unsigned qcap = ntiles + 4u * gridDim.x + 64u;   // > any claim count
  unsigned e_nxt = first_elem(blockIdx.x + gridDim.x);
  unsigned raw = 0;
  bool pend = false;
  if (leader) {
    unsigned w = kNoTile;
    if (e_nxt != kNoTile) w = first_elem(dyn0 + atomic_claim(args.sched, qcap));
    qslot[1] = w;
    pend = w != kNoTile;
    if (pend) raw = atomic_claim(args.sched, qcap);
  }
  cta_sync<TPB>();
  unsigned e_nn = qslot[1];
  fetch_ids(e_nxt, ids_nxt);
  unsigned it = 0;
  auto body = [&](auto BC) {
    constexpr int buf = decltype(BC)::value;
    if (e_nxt != kNoTile) issue(e_nxt, buf ^ 1, ids_nxt);
    cp_async_commit();
    fetch_ids(e_nn, ids_nn);
    if (leader) {
      if (args.l2pf && e_nn != kNoTile) {
        const unsigned b2 = min((unsigned)EPG, e_end - e_nn) * (unsigned)(C * NODES * 8);
        bulk_prefetch_l2(args.u + (size_t)e_nn * (C * NODES), b2);
        if (read_r) bulk_prefetch_l2(gsrc_r + (size_t)e_nn * (C * NODES), b2);
      }
      // publish the claim made one iteration ago, start the next one
      const unsigned w = pend ? first_elem(dyn0 + raw) : kNoTile;
      qslot[buf] = w;
      pend = w != kNoTile;
      if (pend) raw = atomic_claim(args.sched, qcap);
    }
    mbar_wait(&bar[buf], (it >> 1) & 1u);
    cp_async_wait<1>();      // this lane's own face values (it alone reads them)

    double* su = smem + buf * K::BUF;
    double* sr = su + K::TILE;
    const double* snb = su + 2 * K::TILE;
    const unsigned e0 = e_tile;
    const int nel = (int)min((unsigned)EPG, e_end - e0);
    if (plane_lane && (EPG == 1 || q < nel)) {
      const double* mt = su + K::OFF_MAT + q * kMatStride;
      const double ir = mt[0], c2r = mt[1], tau = mt[2], irt = mt[3];
      double* ul = su + q * C * NODES + nb0;
      double* rl = sr + q * C * NODES + nb0;
      double pl[N], vl[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        pl[i] = ul[D * NODES + i * sm];
        vl[i] = ul[M * NODES + i * sm];
      }
      double fv0 = 0.0, fp0 = 0.0, fv1 = 0.0, fp1 = 0.0;
      if (faces) {
        const double* f0 = snb + (((q * D + M) * 2 + 0) * 2) * NF + fn;
        const double* f1 = snb + (((q * D + M) * 2 + 1) * 2) * NF + fn;
        const bool w0 = ids_cur[0] == -1, w1 = ids_cur[1] == -1;
        cart_face_flux(vl[0], pl[0], w0 ? vl[0] : f0[0], w0 ? -pl[0] : f0[NF],
                       geo[GLy::NORMAL + (M * 2 + 0) * D + M], geo[GLy::FSCALE + M * 2 + 0], ir,
                       c2r, tau, irt, stab, fv0, fp0);
        cart_face_flux(vl[N - 1], pl[N - 1], w1 ? vl[N - 1] : f1[0], w1 ? -pl[N - 1] : f1[NF],
                       geo[GLy::NORMAL + (M * 2 + 1) * D + M], geo[GLy::FSCALE + M * 2 + 1], ir,
                       c2r, tau, irt, stab, fv1, fp1);
      }
      const double gmm = geo[M * D + M];
      const double cv = cell ? ir * gmm : 0.0;
      const double cp = cell ? c2r * gmm : 0.0;
      double* ppl = sP + M * (EPG * NODES) + q * NODES + nb0;
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
        ppl[i * sm] = fma(cp, av, fma(l0, fp0, l1 * fp1));
        const int sv = M * NODES + i * sm;
        if (MODE == OUT_MINVK || MODE == OUT_RHS) {
          ul[sv] = MODE == OUT_RHS ? -resv : resv;
        } else if (MODE == OUT_LSRK) {
          const double f = -resv * args.dt;
          const double rr = read_r ? fma(args.a, rl[sv], f) : f;
          rl[sv] = rr;
          ul[sv] = fma(args.b, rr, vl[i]);
        } else if (MODE == OUT_ADERB) {
          rl[sv] = rl[sv] - resv;
        }
      }
    }
    cta_sync<TPB>();       // p shares complete; every group has read the tile's p
    const unsigned e_nnn = qslot[buf];
    // p: the d shares summed in direction order, update, in place
    for (int idx = tid; idx < nel * NODES; idx += TPB) {
      const int q2 = EPG == 1 ? 0 : idx / NODES;
      const int sp = q2 * C * NODES + D * NODES + (idx - q2 * NODES);
      double resp = sP[idx];
#pragma unroll
      for (int m = 1; m < D; ++m) resp = sP[m * (EPG * NODES) + idx] + resp;
      if (MODE == OUT_MINVK || MODE == OUT_RHS) {
        su[sp] = MODE == OUT_RHS ? -resp : resp;
      } else if (MODE == OUT_LSRK) {
        const double f = -resp * args.dt;
        const double rr = read_r ? fma(args.a, sr[sp], f) : f;
        sr[sp] = rr;
        su[sp] = fma(args.b, rr, su[sp]);
      } else if (MODE == OUT_ADERB) {
        sr[sp] = sr[sp] - resp;
      }
    }
    // generic writes of the stage -> visible to the TMA engine, then store
    fence_proxy_async();
    cta_sync<TPB>();
    if (leader) {
      const unsigned tbytes = (unsigned)(nel * C * NODES * 8);
      const size_t goff = (size_t)e0 * (C * NODES);
      auto store = [&](double* g, const double* sm_src) {
        if (WK_L2_HINT) bulk_s2g_hint(g, sm_src, tbytes, pol);
        else bulk_s2g(g, sm_src, tbytes);
      };
      if (MODE == OUT_LSRK) {
        store(args.u_out + goff, su);
        if (!args.r_dead) store(args.r + goff, sr);
      } else if (MODE == OUT_ADERB) {
        store(args.out + goff, sr);
      } else {
        store(args.out + goff, su);
      }
      bulk_commit();
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      ids_cur[s] = ids_nxt[s];
      ids_nxt[s] = ids_nn[s];
    }
    ++it;
    e_tile = e_nxt;
    e_nxt = e_nn;
    e_nn = e_nnn;
  };
  while (true) {
    if (e_tile == kNoTile) break;
    body(std::integral_constant<int, 0>{});
    if (e_tile == kNoTile) break;
    body(std::integral_constant<int, 1>{});
  }
  if (M == 0) {
    sched_done(args.sched, leader, pend, raw);
    if (leader) bulk_wait<0>();
  }
}

template <int D, int N, int MODE, bool FAST>
__global__ void __launch_bounds__(StreamDCfg<D, N>::TPB, StreamDCfg<D, N>::MINB)
affine_streamd_kernel(const AffineArgs args) {
  using K = StreamDCfg<D, N>;
  extern __shared__ __align__(128) double smem[];
  WK_CHECK_SMEM(K::BYTES);
  const int tid = threadIdx.x;
  for (int i = tid; i < GeoLayout<D>::STRIDE; i += K::TPB) smem[K::OFF_GEO + i] = args.geo[i];
  if (tid == 0) {
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + K::OFF_BAR);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int g = tid / K::TG;
  if (g == 0) {
    streamd_run<D, N, MODE, FAST, 0>(args, smem);
  } else if (g == 1) {
    streamd_run<D, N, MODE, FAST, 1>(args, smem);
  } else if (D == 3) {
    streamd_run<D, N, MODE, FAST, (D == 3 ? 2 : 1)>(args, smem);
  }
}

}  // namespace wk
