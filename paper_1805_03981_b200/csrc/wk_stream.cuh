// Persistent streaming version of the Cartesian pencil operator (the LSRK
// stage / rhs / M^{-1}K / ADER-B hot path of configs 1, 2, 4, 5).
//
// Arithmetic and pencil mapping are those of affine_group_kernel
// (wk_group.cuh): a group of TG threads owns EPG elements, lane = pencil, the
// two face integrands of a pencil are computed by that lane, v_m is finished
// per direction and p after the last one.  What changes is the schedule:
//
//  * one group per CTA, persistent over tiles t = blockIdx.x + k * gridDim.x;
//  * two shared-memory stages per group.  While tile t is computed, tile
//    t+grid streams in: the u and r (or V) tiles with ONE cp.async.bulk (TMA)
//    each, completion on an mbarrier with expect_tx; the neighbour face
//    values (v_m and p at both ends of each pencil) with 8-byte cp.async;
//  * neighbour ids are fetched one tile earlier still.
// Every warp therefore always has its next tile's bytes in flight, and the
// per-element staging shrinks to two TMA instructions plus the face gathers.
#pragma once
#include "wk_group.cuh"

namespace wk {

// End of a tile-queue kernel: wait for lane 0's last claim, count this CTA
// as done; the last CTA resets both counters for the next launch (every
// claim of this launch has returned by then).
__device__ __forceinline__ void sched_done(unsigned* sched, bool leader, bool pend, unsigned raw) {
  if (!leader) return;
  if (pend && raw == 0xFFFFFFFFu) __trap();   // consumes the claim's result
  __threadfence();
  if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
    atomicExch(sched, 0u);
    atomicExch(sched + 1, 0u);
    __threadfence();
  }
}

template <int D, int N>
struct StreamCfg {
  using G = GroupCfg<D, N>;
  static constexpr int C = D + 1, NODES = G::NODES, NF = G::NF, EPG = G::EPG, TG = G::TG;
  static constexpr int TILE = EPG * C * NODES;
  static constexpr int NBF = EPG * D * 2 * 2 * NF;       // [q][m][side][v_m,p][fn]
  static constexpr int BUF = (2 * TILE + NBF + 1) / 2 * 2;
  static constexpr int OFF_RP = 2 * BUF;
  static constexpr int OFF_BAR = (OFF_RP + EPG * NODES + 1) / 2 * 2;
  static constexpr int OFF_Q = OFF_BAR + 2;              // two 8-byte mbarriers
  static constexpr int OFF_TAB = OFF_Q + 4;              // two tile-queue slots + elements
  static constexpr int TOTAL = OFF_TAB + N * N + 2 * N + GeoLayout<D>::STRIDE;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  static constexpr bool TILE16 = (TILE * 8) % 16 == 0;
};

template <int D, int N, int MODE>
__global__ void __launch_bounds__(StreamCfg<D, N>::TG)
affine_stream_kernel(const AffineArgs args) {
  using K = StreamCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, EPG = K::EPG, TG = K::TG;
  constexpr bool READ_RV = (MODE == OUT_LSRK) || (MODE == OUT_ADERB);
  extern __shared__ __align__(128) double smem[];
  double* const srp = smem + K::OFF_RP;
  unsigned long long* const bar = reinterpret_cast<unsigned long long*>(smem + K::OFF_BAR);
  double* const geo = smem + K::OFF_TAB + N * N + 2 * N;
  const int lane = threadIdx.x;
  WK_CHECK_SMEM(K::BYTES);
  // r / V in and every result out: L2 evict_first (wk_common.cuh)
  const unsigned long long pol = lane == 0 ? l2_evict_first_policy() : 0ull;
  for (int i = lane; i < GLy::STRIDE; i += TG) geo[i] = args.geo[i];
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  group_sync<TG>(0);

  const bool faces = (args.parts & PART_FACE) != 0;
  const bool cell = (args.parts & PART_CELL) != 0;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || args.a != 0.0);
  const double* __restrict__ gsrc_r = (MODE == OUT_ADERB) ? args.v : args.r;
  const long long e_end = args.e_begin + args.E;
  const long long ntiles = (args.E + EPG - 1) / EPG;
  // TMA path needs 16-byte aligned tile starts (all tiles, so e_begin too)
  const bool tma = K::TILE16 && (((args.e_begin * C * NODES) & 1) == 0);
  const int q = lane / NF, fn = lane - (lane / NF) * NF;
  const bool plane_lane = lane < EPG * NF;

  long long tile = blockIdx.x;
  if (tile >= ntiles) return;
  // lane-constant offsets: neighbour face node per (m, side); this lane's
  // face-value slots in both stages
  int noff[D][2];
#pragma unroll
  for (int m = 0; m < D; ++m)
#pragma unroll
    for (int s = 0; s < 2; ++s) noff[m][s] = face_to_node<N>(m, 1 - s, fn);
  unsigned nb_u32[2];
#pragma unroll
  for (int b = 0; b < 2; ++b)
    nb_u32[b] = smem_u32(smem + b * K::BUF + 2 * K::TILE + (q * D * 2 * 2) * NF + fn);
  // the collapsed 1-D tables in registers for the whole kernel
  double rA[N * N], rL0[N], rL1[N];
#pragma unroll
  for (int i = 0; i < N * N; ++i) rA[i] = args.cA[i];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    rL0[i] = args.cL0[i];
    rL1[i] = args.cL1[i];
  }

  auto fetch_ids = [&](long long t, long long et, int (&ids)[2 * D]) {
    const long long e = et + q;
#pragma unroll
    for (int f = 0; f < 2 * D; ++f)
      ids[f] = (faces && plane_lane && t < ntiles && e < e_end)
                   ? __ldg(args.nbr + e * 2 * D + f) : -1;
  };
  auto issue = [&](long long et, int b, const int (&ids)[2 * D]) {
    const long long e0 = et;
    const int nel = (int)min((long long)EPG, e_end - e0);
    double* su = smem + b * K::BUF;
    double* sr = su + K::TILE;
    double* snb = su + 2 * K::TILE;
    const unsigned bytes = (unsigned)(nel * C * NODES * 8);
    const double* gu = args.u + e0 * C * NODES;
    const double* gr = gsrc_r + e0 * C * NODES;
    if (tma && (bytes % 16) == 0) {
      if (lane == 0) {
        bulk_wait_read<0>();   // earlier bulk stores from this stage have read it
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[b], read_r ? 2 * bytes : bytes);
        bulk_g2s(su, gu, bytes, &bar[b]);
        if (read_r) bulk_g2s_hint(sr, gr, bytes, &bar[b], pol);
      }
    } else {
      if (lane == 0) bulk_wait_read<0>();
      group_sync<TG>(0);
      for (int i = lane; i < nel * C * NODES; i += TG) {
        cp_async8(su + i, gu + i);
        if (read_r) cp_async8(sr + i, gr + i);
      }
      if (lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar[b]))
                     : "memory");
      }
    }
    if (faces && plane_lane && q < nel) {
      const unsigned dst = nb_u32[b];
#pragma unroll
      for (int m = 0; m < D; ++m)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int nb = ids[2 * m + s];
          WK_CHECK_NBR(args, nb);
          const unsigned d0 = dst + (unsigned)(((m * 2 + s) * 2) * NF) * 8u;
          if (nb >= 0) {
            const double* src = args.u + (long long)nb * (C * NODES) + noff[m][s];
            cp_async8_u32(d0, src + m * NODES);
            cp_async8_u32(d0 + NF * 8u, src + D * NODES);
          } else if (args.has_ghost && nb <= -2) {
            const double* src = args.ghost + (long long)ghost_slot(nb) * C * NF + fn;
            cp_async8_u32(d0, src + m * NF);
            cp_async8_u32(d0 + NF * 8u, src + D * NF);
          }
        }
    }
  };

  auto fetch_mat = [&](long long t, long long et, double (&mt)[4]) {
    const long long e = et + q;
    const bool ok = plane_lane && t < ntiles && e < e_end;
#pragma unroll
    for (int i = 0; i < 4; ++i) mt[i] = ok ? __ldg(args.mat + e * kMatStride + i) : 0.0;
  };
  int ids_cur[2 * D], ids_nxt[2 * D], ids_nn[2 * D];
  double mat_cur[4], mat_nxt[4];
  long long e_tile = tile_elem<EPG>(args, tile);
  fetch_ids(tile, e_tile, ids_cur);
  fetch_mat(tile, e_tile, mat_cur);
  issue(e_tile, 0, ids_cur);
  cp_async_commit();
  // Tile queue.  A CTA's first two tiles are static (blockIdx.x, +grid);
  // every later one is claimed from a global counter (args.sched[0]) two
  // iterations before it is computed.  Tiles are therefore taken in mesh
  // order and the tiles in flight form ONE compact window: the neighbour
  // faces a tile gathers were just streamed in by the CTAs working next to
  // it and hit in L2 (a static round-robin lets CTAs drift apart, and the
  // face gathers then re-read DRAM: +75 % read traffic at config 5).  The
  // last CTA to finish resets the counters for the next launch.
  long long* const qslot = reinterpret_cast<long long*>(smem + K::OFF_Q);
  const long long kNone = ntiles;                 // "no more work"
  const long long dyn0 = 2LL * gridDim.x;
  const unsigned qcap = (unsigned)(ntiles + 4LL * gridDim.x + 64);   // > any claim count         // first dynamically claimed tile
  long long nxt = tile + gridDim.x < ntiles ? tile + gridDim.x : kNone;
  long long e_nxt = nxt < ntiles ? tile_elem<EPG>(args, nxt) : 0;
  unsigned raw = 0;                               // lane 0: claim in flight
  bool pend = false;
  if (lane == 0) {
    long long w = kNone;
    if (nxt < ntiles) {
      w = dyn0 + (long long)atomic_claim(args.sched, qcap);
      if (w >= ntiles) w = kNone;
    }
    qslot[1] = w;
    qslot[3] = w < ntiles ? tile_elem<EPG>(args, w) : 0;   // its first element
    pend = w < ntiles;
    if (pend) raw = atomic_claim(args.sched, qcap);
  }
  group_sync<TG>(0);
  long long nn = qslot[1], e_nn = qslot[3];
  fetch_ids(nxt, e_nxt, ids_nxt);
  int buf = 0;
  unsigned it = 0;
  while (tile < ntiles) {
    if (nxt < ntiles) issue(e_nxt, buf ^ 1, ids_nxt);
    cp_async_commit();
    fetch_ids(nn, e_nn, ids_nn);
    fetch_mat(nxt, e_nxt, mat_nxt);
    if (tma && args.l2pf && lane == 0 && nn < ntiles) {
      // two tiles ahead: into L2 only, so more DRAM reads are in flight than
      // the two shared-memory stages hold
      const long long e2 = e_nn;
      const unsigned b2 = (unsigned)(min((long long)EPG, e_end - e2) * C * NODES * 8) & ~15u;
      bulk_prefetch_l2(args.u + e2 * C * NODES, b2);
      if (read_r) bulk_prefetch_l2(gsrc_r + e2 * C * NODES, b2);
    }
    if (lane == 0) {
      // publish the claim made one iteration ago, start the next one
      long long w = kNone;
      if (pend) {
        w = dyn0 + (long long)raw;
        if (w >= ntiles) w = kNone;
      }
      qslot[it & 1] = w;
      qslot[2 + (it & 1)] = w < ntiles ? tile_elem<EPG>(args, w) : 0;
      pend = w < ntiles;
      if (pend) raw = atomic_claim(args.sched, qcap);
    }
    mbar_wait(&bar[buf], (it >> 1) & 1u);
    cp_async_wait<1>();
    group_sync<TG>(0);
    const long long nnn = qslot[it & 1], e_nnn = qslot[2 + (it & 1)];

    double* su = smem + buf * K::BUF;
    double* sr = su + K::TILE;
    const double* snb = su + 2 * K::TILE;
    const long long e0 = e_tile;
    const int nel = (int)min((long long)EPG, e_end - e0);
    // results go back into the stage (u_out / out over u, r over r) and leave
    // with one bulk store per tile, unless the tile is not TMA-aligned
    const unsigned tbytes = (unsigned)(nel * C * NODES * 8);
    const bool bstore = tma && (tbytes % 16) == 0;
    const bool plane = plane_lane && q < nel;
    const long long e = e0 + q;
    const double ir = mat_cur[0], c2r = mat_cur[1], tau = plane ? mat_cur[2] : 1.0,
                 irt = mat_cur[3];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
      if (plane) {
        const int nb0 = pencil_base<N>(m, fn);
        const long long gbase = e * C * NODES + nb0;
        double* ul = su + q * C * NODES + nb0;
        double* rl = sr + q * C * NODES + nb0;
        double pl[N], vl[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          pl[i] = ul[D * NODES + i * sm];
          vl[i] = ul[m * NODES + i * sm];
        }
        double fv0 = 0.0, fp0 = 0.0, fv1 = 0.0, fp1 = 0.0;
        if (faces) {
          const double* f0 = snb + (((q * D + m) * 2 + 0) * 2) * NF + fn;
          const double* f1 = snb + (((q * D + m) * 2 + 1) * 2) * NF + fn;
          const bool w0 = ids_cur[2 * m] == -1, w1 = ids_cur[2 * m + 1] == -1;
          cart_face_flux(vl[0], pl[0], w0 ? vl[0] : f0[0], w0 ? -pl[0] : f0[NF],
                         geo[GLy::NORMAL + (m * 2 + 0) * D + m], geo[GLy::FSCALE + m * 2 + 0],
                         ir, c2r, tau, irt, args.stab, fv0, fp0);
          cart_face_flux(vl[N - 1], pl[N - 1], w1 ? vl[N - 1] : f1[0],
                         w1 ? -pl[N - 1] : f1[NF], geo[GLy::NORMAL + (m * 2 + 1) * D + m],
                         geo[GLy::FSCALE + m * 2 + 1], ir, c2r, tau, irt, args.stab, fv1,
                         fp1);
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
            const double a = rA[i * N + j];
            ap = fma(a, pl[j], ap);
            av = fma(a, vl[j], av);
          }
          const double l0 = rL0[i], l1 = rL1[i];
          const double resv = fma(cv, ap, fma(l0, fv0, l1 * fv1));
          double resp = fma(cp, av, fma(l0, fp0, l1 * fp1));
          if (m > 0) resp += rpl[i * sm];
          const long long iv = gbase + m * NODES + i * sm;
          const int sv = m * NODES + i * sm;      // smem offsets in the element tile
          const int spn = D * NODES + i * sm;
          if (MODE == OUT_MINVK || MODE == OUT_RHS) {
            const double o = MODE == OUT_RHS ? -resv : resv;
            if (bstore) ul[sv] = o; else args.out[iv] = o;
          } else if (MODE == OUT_LSRK) {
            const double f = -resv * args.dt;
            const double rr = read_r ? fma(args.a, rl[sv], f) : f;
            const double un = fma(args.b, rr, vl[i]);
            if (bstore) {
              rl[sv] = rr;
              ul[sv] = un;
            } else {
              args.r[iv] = rr;
              args.u_out[iv] = un;
            }
          } else if (MODE == OUT_ADERB) {
            const double o = rl[sv] - resv;
            if (bstore) rl[sv] = o; else args.out[iv] = o;
          }
          if (m < D - 1) {
            rpl[i * sm] = resp;
          } else {
            const long long ip = gbase + D * NODES + i * sm;
            if (MODE == OUT_MINVK || MODE == OUT_RHS) {
              const double o = MODE == OUT_RHS ? -resp : resp;
              if (bstore) ul[spn] = o; else args.out[ip] = o;
            } else if (MODE == OUT_LSRK) {
              const double f = -resp * args.dt;
              const double rr = read_r ? fma(args.a, rl[spn], f) : f;
              const double un = fma(args.b, rr, pl[i]);
              if (bstore) {
                rl[spn] = rr;
                ul[spn] = un;
              } else {
                args.r[ip] = rr;
                args.u_out[ip] = un;
              }
            } else if (MODE == OUT_ADERB) {
              const double o = rl[spn] - resp;
              if (bstore) rl[spn] = o; else args.out[ip] = o;
            }
          }
        }
      }
      group_sync<TG>(0);   // p shares visible to the next direction / stage reusable
    }
    if (bstore) {
      // make this stage's generic writes visible to the TMA engine, then store
      fence_proxy_async();
      group_sync<TG>(0);
      if (lane == 0) {
        const long long goff = e0 * C * NODES;
        if (MODE == OUT_LSRK) {
          bulk_s2g_hint(args.u_out + goff, su, tbytes, pol);
          if (!args.r_dead) bulk_s2g_hint(args.r + goff, sr, tbytes, pol);
        } else if (MODE == OUT_ADERB) {
          bulk_s2g_hint(args.out + goff, sr, tbytes, pol);
        } else {
          bulk_s2g_hint(args.out + goff, su, tbytes, pol);
        }
        bulk_commit();
      }
    }
#pragma unroll
    for (int f = 0; f < 2 * D; ++f) {
      ids_cur[f] = ids_nxt[f];
      ids_nxt[f] = ids_nn[f];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) mat_cur[i] = mat_nxt[i];
    buf ^= 1;
    ++it;
    tile = nxt;
    nxt = nn;
    nn = nnn;
    e_tile = e_nxt;
    e_nxt = e_nn;
    e_nn = e_nnn;
  }
  sched_done(args.sched, lane == 0, pend, raw);
  if (lane == 0) bulk_wait<0>();
}

}  // namespace wk
