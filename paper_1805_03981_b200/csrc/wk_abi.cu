// extern "C" entry points (include/wavekernel_b200.h): context lifecycle,
// host-built tables and programs, kernel dispatch over (d, n).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/wavekernel_b200.h"
#include "wk_basis.h"
#include "wk_error.h"
#include "wk_generic.cuh"
#include "wk_launch.h"
#include "wk_fields.cuh"

using namespace wk;

namespace {

thread_local std::string g_err;

std::vector<double> to_double(const Mat& m) { return std::vector<double>(m.begin(), m.end()); }

template <typename T>
T* upload(const T* host, size_t count) {
  T* d = nullptr;
  if (count == 0) return nullptr;
  WK_CUDA(cudaMalloc(&d, count * sizeof(T)));
  WK_CUDA(cudaMemcpy(d, host, count * sizeof(T), cudaMemcpyDefault));   // host or device source
  return d;
}

int reduction_stride(int policy) {
  require(policy >= 0 && policy <= 3, "unknown degree-reduction policy");
  return policy;
}

// reduction_schedule (kernels.py:286-302)
std::vector<std::pair<int, int>> schedule(int k, int policy) {
  const int s = reduction_stride(policy);
  std::vector<std::pair<int, int>> out;
  int deg = k;
  for (int j = 1; j <= k + 1; ++j) {
    int nxt = (s && j % s == 0) ? std::max(deg - s, 0) : deg;
    out.push_back({deg, nxt});
    deg = nxt;
  }
  return out;
}

double taylor_weight(int j, double dt) {  // stepping.py:210-212
  double f = 1.0;
  for (int i = 2; i <= j + 1; ++i) f *= i;
  double p = 1.0;
  for (int i = 0; i < j + 1; ++i) p *= dt;
  return (j % 2 ? -1.0 : 1.0) * p / f;
}

}  // namespace

// ---------------------------------------------------------------------------
namespace wk {
int num_sms() {
  int dev = 0, sms = 0;
  WK_CUDA(cudaGetDevice(&dev));
  WK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

KernelSetup& kernel_setup(const void* kernel) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, KernelSetup> cache;
  int dev = 0;
  WK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  return cache[{dev, kernel}];   // std::map: references stay valid
}

// 1-D tables
Mat table_B(int k) { return lagrange(gl_nodes(k), g_nodes(k), false); }
Mat table_Binv(int k) { return lagrange(g_nodes(k), gl_nodes(k), false); }
Mat table_Dgl(int k) { return lagrange(gl_nodes(k), g_nodes(k), true); }
Mat table_Dco(int k) { return lagrange(g_nodes(k), g_nodes(k), true); }
Mat table_Dglco(int k) { return lagrange(gl_nodes(k), gl_nodes(k), true); }
std::vector<long double> gauss_w(int k) {
  std::vector<long double> x, w;
  gauss_rule(k + 1, x, w);
  return w;
}
Mat table_M1(int k) {  // B^T W B
  const int n = k + 1;
  Mat B = table_B(k), WB = B;
  auto w = gauss_w(k);
  for (int q = 0; q < n; ++q)
    for (int j = 0; j < n; ++j) WB[q * n + j] *= w[q];
  return matmul(transpose(B, n, n), WB, n, n, n);
}
Mat table_BtW(int k) {  // B^T W  (from_gauss_weighted on affine cells)
  const int n = k + 1;
  Mat Bt = transpose(table_B(k), n, n);
  auto w = gauss_w(k);
  for (int j = 0; j < n; ++j)
    for (int q = 0; q < n; ++q) Bt[j * n + q] *= w[q];
  return Bt;
}
// A = 1/2 M1^{-1} (B^T W Dgl - Dgl^T W B): split strong/weak cell operator
Mat table_A(int k) {
  const int n = k + 1;
  Mat B = table_B(k), Dg = table_Dgl(k);
  auto w = gauss_w(k);
  Mat WB = B, WD = Dg;
  for (int q = 0; q < n; ++q)
    for (int j = 0; j < n; ++j) {
      WB[q * n + j] *= w[q];
      WD[q * n + j] *= w[q];
    }
  Mat s1 = matmul(transpose(B, n, n), WD, n, n, n);
  Mat s2 = matmul(transpose(Dg, n, n), WB, n, n, n);
  Mat diff(n * n);
  for (int i = 0; i < n * n; ++i) diff[i] = 0.5L * (s1[i] - s2[i]);
  return matmul(inverse(table_M1(k), n), diff, n, n, n);
}
Mat table_lift(int k) {  // rows: M1^{-1} e_0, M1^{-1} e_{n-1}
  const int n = k + 1;
  Mat mi = inverse(table_M1(k), n), out(2 * n);
  for (int i = 0; i < n; ++i) {
    out[i] = mi[i * n + 0];
    out[n + i] = mi[i * n + (n - 1)];
  }
  return out;
}
}  // namespace wk

// ---------------------------------------------------------------------------
struct TckProgram {
  int* d_ops = nullptr;
  double* d_tab = nullptr;
  int nops = 0, tab_len = 0, acc_len = 0;
  std::vector<double> enc;     // weight code per op: <0 -> Taylor index -(1+j)
  std::vector<int> h_ops;      // host copies for the compile-time-plan kernel
  std::vector<double> h_tab;
  int plan_ok = -1;            // -1 unchecked, 0/1: matches make_tck_plan
};

struct wk_ctx {
  int D = 0, k = 0, N = 0, C = 0, NODES = 0, NF = 0;
  long long E = 0, G = 0;
  int stab = 1, mode = WK_GEOM_AFFINE, cart = 0;
  int* d_nbr = nullptr;
  double* d_mat = nullptr;
  double* d_geo = nullptr;
  int* d_cls = nullptr;
  long long n_classes = 0;
  double* d_ghost = nullptr;
  bool own_ghost = true;
  double* d_optab = nullptr;  // A, L0, L1
  std::vector<double> h_optab;
  std::map<std::string, double*> tables;
  double* scratch = nullptr;
  std::map<int, TckProgram> progs;
  long long n_export = 0;
  long long* d_exp_elem = nullptr;
  int* d_exp_face = nullptr;
  long long range_begin = 0, range_count = -1;
  long long tord_ch = 0, tord_ns = 0, tord_nb = 0;   // structured traversal (wk_set_tile_order)
  unsigned* d_sched = nullptr;  // tile-queue counters (zero; reset by each launch's last CTA)
  int queue_slot = 0;           // counter pair of the next launches (concurrent streams)
  // curved geometry
  std::map<int, double*> d_invjac, d_jxw;
  double* d_fnormal[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double* d_fjxw[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double* d_ctab = nullptr;  // curved tables: B, Binv, Dco, DcoT, BT
  double* d_crec = nullptr;  // curved per-element metric records (wk_stream_curved.cuh)
  std::vector<double> h_ctab;
  std::vector<double*> owned;

  double* table(const std::string& key, const Mat& m) {
    auto it = tables.find(key);
    if (it != tables.end()) return it->second;
    auto v = to_double(m);
    double* d = upload(v.data(), v.size());
    tables[key] = d;
    return d;
  }
  double* scratch_buf() {
    if (!scratch) WK_CUDA(cudaMalloc(&scratch, sizeof(double) * (size_t)E * C * NODES));
    return scratch;
  }
  double* d_part = nullptr;     // per-element partial sums (state norm)
  double* part_buf() {
    if (!d_part) {
      WK_CUDA(cudaMalloc(&d_part, sizeof(double) * (size_t)(E > 0 ? E : 1)));
      owned.push_back(d_part);
    }
    return d_part;
  }
  long long rbegin() const { return range_count < 0 ? 0 : range_begin; }
  long long rcount() const { return range_count < 0 ? E : range_count; }
};

namespace {

// ---- curved-geometry glue (kernels in wk_curved.cuh) ---------------------
CurvedArgs curved_args(wk_ctx* c) {
  CurvedArgs a{};
  if (c->mode != WK_GEOM_CURVED) return a;
  a.inv_jac = c->d_invjac.at(c->k);
  a.jxw = c->d_jxw.at(c->k);
  for (int f = 0; f < 2 * c->D; ++f) {
    a.fnormal[f] = c->d_fnormal[f];
    a.fjxw[f] = c->d_fjxw[f];
  }
  a.ctab = c->d_ctab;
  for (auto& kv : c->d_invjac) a.invjac_deg[kv.first] = kv.second;
  return a;
}

void curved_setup(wk_ctx* c, const wk_desc* desc) {
  require(desc->n_curved_degrees >= 1 && desc->curved_degrees[0] == desc->degree,
          "curved geometry needs the degree-k point set first");
  require(c->N <= 8, "curved geometry supports degrees up to 7");
  const long long E = c->E;
  const int D = c->D;
  for (int i = 0; i < desc->n_curved_degrees; ++i) {
    const int q = desc->curved_degrees[i];
    require(q >= 0 && q <= c->k, "curved degree out of range");
    const size_t np = D == 3 ? (size_t)(q + 1) * (q + 1) * (q + 1) : (size_t)(q + 1) * (q + 1);
    c->d_invjac[q] = upload(desc->curved_inv_jac[i], (size_t)E * D * D * np);
    c->d_jxw[q] = upload(desc->curved_jxw[i], (size_t)E * np);
    c->owned.push_back(c->d_invjac[q]);
    c->owned.push_back(c->d_jxw[q]);
  }
  for (int f = 0; f < 2 * D; ++f) {
    c->d_fnormal[f] = upload(desc->face_normal[f], (size_t)E * D * c->NF);
    c->d_fjxw[f] = upload(desc->face_jxw[f], (size_t)E * c->NF);
    c->owned.push_back(c->d_fnormal[f]);
    c->owned.push_back(c->d_fjxw[f]);
  }
  const int n = c->N;
  Mat B = table_B(c->k), Binv = table_Binv(c->k), Dco = table_Dco(c->k);
  Mat all;
  for (const Mat* m : {&B, &Binv, &Dco}) all.insert(all.end(), m->begin(), m->end());
  Mat DcoT = transpose(Dco, n, n), BT = transpose(B, n, n);
  all.insert(all.end(), DcoT.begin(), DcoT.end());
  all.insert(all.end(), BT.begin(), BT.end());
  auto v = to_double(all);
  c->d_ctab = upload(v.data(), v.size());
  c->h_ctab = v;
  c->owned.push_back(c->d_ctab);
  if (stream_curved_supported(D, n) && E > 0) {
    // per-element records for the streaming kernels: one strided 2-D copy
    // per array into (E, len) with the record's offsets
    const int nodes = n * n * n, nf = n * n, len = crec_len(n);
    auto ev = [](int x) { return (x + 1) / 2 * 2; };
    WK_CUDA(cudaMalloc(&c->d_crec, sizeof(double) * (size_t)E * len));
    c->owned.push_back(c->d_crec);
    auto put = [&](int off, const double* src, int cnt) {
      WK_CUDA(cudaMemcpy2D(c->d_crec + off, sizeof(double) * len, src, sizeof(double) * cnt,
                           sizeof(double) * cnt, (size_t)E, cudaMemcpyDeviceToDevice));
    };
    int off = 0;
    put(off, c->d_invjac.at(c->k), 9 * nodes);
    off += ev(9 * nodes);
    put(off, c->d_jxw.at(c->k), nodes);
    off += ev(nodes);
    for (int f = 0; f < 6; ++f) put(off + f * 3 * nf, c->d_fnormal[f], 3 * nf);
    off += ev(18 * nf);
    for (int f = 0; f < 6; ++f) put(off + f * nf, c->d_fjxw[f], nf);
  }
}

// persistent curved kernels: per-element arrays + the 1-D tables by value
CurvedStreamArgs curved_stream_args(wk_ctx* c) {
  CurvedStreamArgs a{};
  a.rec = c->d_crec;
  for (auto& kv : c->d_invjac)
    if (kv.first >= 0 && kv.first < kMaxN) a.inv_jac[kv.first] = kv.second;
  a.jxw = c->d_jxw.at(c->k);
  for (int f = 0; f < 2 * c->D; ++f) {
    a.fnormal[f] = c->d_fnormal[f];
    a.fjxw[f] = c->d_fjxw[f];
  }
  for (size_t i = 0; i < c->h_ctab.size() && i < (size_t)kCTab; ++i) a.ctab[i] = c->h_ctab[i];
  return a;
}

// ---- affine operator launch --------------------------------------------
AffineArgs affine_args(wk_ctx* c) {
  AffineArgs a{};
  a.nbr = c->d_nbr;
  a.ghost = c->d_ghost;
  a.geo = c->d_geo;
  a.geo_class = c->d_cls;
  a.mat = c->d_mat;
  a.tab = c->d_optab;
  {
    const int n = c->N;
    for (int i = 0; i < n * n; ++i) a.cA[i] = c->h_optab[i];
    for (int i = 0; i < n; ++i) {
      a.cL0[i] = c->h_optab[n * n + i];
      a.cL1[i] = c->h_optab[n * n + n + i];
    }
  }
  a.E = c->rcount();
  a.e_begin = c->rbegin();
  a.e_total = c->E;
  a.n_ghost = c->G;
  // structured traversal of full-mesh launches (range launches keep mesh order)
  a.tmap_ch = a.tmap_ns = a.tmap_nb = 0;
  if (c->tord_ch > 0 && c->range_count < 0 &&
      (unsigned long long)c->E * (unsigned long long)c->tord_ch < (1ull << 32) &&
      (unsigned long long)c->E * (unsigned long long)c->tord_ns < (1ull << 32)) {
    a.tmap_ch = (unsigned)c->tord_ch;
    a.tmap_ns = (unsigned)c->tord_ns;
    a.tmap_nb = (unsigned)c->tord_nb;
    a.tmap_ch_m = a.tmap_ch > 1 ? 0xFFFFFFFFu / a.tmap_ch + 1u : 0u;
    a.tmap_ns_m = a.tmap_ns > 1 ? 0xFFFFFFFFu / a.tmap_ns + 1u : 0u;
  }
  a.parts = PART_BOTH;
  a.stab = c->stab;
  a.has_ghost = c->G > 0 ? 1 : 0;
  a.sched = c->d_sched + 2 * c->queue_slot;
  // An interior-range launch on queue slot 0 runs while the halo stream packs,
  // exchanges (NCCL's kernels need SM slots too) and launches the boundary
  // range: leave kHoldSMs SMs' worth of CTA slots free so that work is not
  // queued behind the persistent grid.  Measured neutral for the interior
  // itself (32^3 slab, P = 2: 0.461 ms/step with 0 SMs held, 0.463 with 8;
  // c5 / 8: 1.953 -> 1.961).  WK_GRID_HOLD overrides.
  {
    constexpr int kHoldSMs = 8;
    static int env = -2;
    if (env == -2) {
      const char* e = getenv("WK_GRID_HOLD");
      env = e ? atoi(e) : -1;
    }
    const bool interior = c->range_count >= 0 && c->queue_slot == 0 && c->G > 0;
    a.grid_hold = interior ? (env >= 0 ? env : kHoldSMs) : 0;
  }
  // The L2 prefetch pays while the working set is within a few L2 sizes
  // (config 2: 0.43 -> 0.49 ms/step without it; config 4's 1.8 GB vectors:
  // 7.7 -> 8.8 ms) and costs once it is far beyond (config 5's 4.2 GB
  // vectors: 15.8 -> 18.6 ms with it).  With the small tiles of n <= 6 it
  // already costs at 0.5 GB vectors (config 5 x-slabs, LSRK45 per rank:
  // 1/2 of the mesh 9.58 -> 7.78 ms, 1/4 4.27 -> 3.77, 1/8 2.37 -> 1.96
  // without it) while the 131 MB vectors of config 2 still gain (a 32^3
  // slab: 0.523 -> 0.459 ms with it).  WK_L2PF=0/1 overrides.
  {
    static int env = -2;
    if (env == -2) {
      const char* e = getenv("WK_L2PF");
      env = e ? atoi(e) : -1;
    }
    const double vec_bytes = 8.0 * (double)c->E * c->C * c->NODES;
    const double limit = c->N >= 7 ? 2.5e9 : 2.6e8;
    a.l2pf = env >= 0 ? env : (vec_bytes <= limit ? 1 : 0);
  }
  return a;
}

template <int D, int N>
struct AffineOp {
  static void run(wk_ctx* c, int mode, const AffineArgs& a, cudaStream_t s) {
    affine_op_launch<D, N>(c->cart != 0, mode, a, s);
  }
};
template <int D, int N>
struct AderA {
  static void run(wk_ctx* c, bool hdg, const TckArgs& a, cudaStream_t s) {
    affine_ader_a_launch<D, N>(c->cart != 0, hdg, a, s);
  }
};
template <int D, int N>
struct StreamAderA {
  static void run(bool hdg, int stride, bool shift, const TckStreamArgs& a, cudaStream_t s,
                  bool& done) {
    done = affine_stream_ader_launch<D, N>(hdg, stride, shift, a, s);
  }
};
template <int D, int N>
struct CurvedStream {
  static void run(int kind, int stride, bool shift, const CurvedStreamArgs& a, cudaStream_t s,
                  bool& done) {
    done = curved_stream_launch<D, N>(kind, stride, shift, a, s);
  }
};
// WK_ADER_KERNEL=group selects the run-time-interpreted ADER kernel A
bool stream_ader_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("WK_ADER_KERNEL");
    on = (e && std::string(e) == "group") ? 0 : 1;
  }
  return on == 1;
}
template <int D, int N>
struct CurvedOp {
  static void run(int mode, const AffineArgs& a, const CurvedArgs& g, cudaStream_t s) {
    curved_op_launch<D, N>(mode, a, g, s);
  }
};
template <int D, int N>
struct CurvedAderA {
  static void run(bool hdg, const TckArgs& a, const CurvedArgs& g, cudaStream_t s) {
    curved_ader_a_launch<D, N>(hdg, a, g, s);
  }
};

template <template <int, int> class F, typename... Args>
void dispatch_dn(int D, int N, Args&&... args) {
#define WK_CASE(d, n) \
  case d * 16 + n:    \
    return F<d, n>::run(std::forward<Args>(args)...);
  switch (D * 16 + N) {
    WK_CASE(2, 2) WK_CASE(2, 3) WK_CASE(2, 4) WK_CASE(2, 5) WK_CASE(2, 6) WK_CASE(2, 7)
    WK_CASE(2, 8) WK_CASE(2, 9) WK_CASE(3, 2) WK_CASE(3, 3) WK_CASE(3, 4) WK_CASE(3, 5)
    WK_CASE(3, 6) WK_CASE(3, 7) WK_CASE(3, 8) WK_CASE(3, 9)
  }
#undef WK_CASE
  throw WkError(WK_EINVAL, "unsupported (dim, degree)");
}

void run_op(wk_ctx* c, int mode, AffineArgs a, cudaStream_t s) {
  if (c->mode == WK_GEOM_AFFINE) {
    dispatch_dn<AffineOp>(c->D, c->N, c, mode, a, s);
  } else {
    if (stream_curved_supported(c->D, c->N) && stream_ader_enabled() && a.parts == PART_BOTH &&
        (mode == OUT_MINVK || mode == OUT_RHS || mode == OUT_LSRK || mode == OUT_ADERB)) {
      CurvedStreamArgs ca = curved_stream_args(c);
      ca.t.op = a;
      bool done = false;
      dispatch_dn<CurvedStream>(c->D, c->N, mode, 0, false, ca, s, done);
      if (done) return;
    }
    dispatch_dn<CurvedOp>(c->D, c->N, mode, a, curved_args(c), s);
  }
}

// generic sweep launch: out = out_scale * post(M^{(x)d} pre(in))
void sweep(wk_ctx* c, const double* in, double* out, const double* dmat, int nf, int nt,
           int pre, int post, const double* pts, double out_scale, cudaStream_t s) {
  SweepArgs a{};
  a.in = in;
  a.out = out;
  a.mat = dmat;
  a.pts = pts;
  a.geo = c->d_geo;
  a.geo_class = c->d_cls;
  a.geo_stride = c->D == 3 ? GeoLayout<3>::STRIDE : GeoLayout<2>::STRIDE;
  a.det_off = c->D == 3 ? GeoLayout<3>::DET : GeoLayout<2>::DET;
  a.E = c->E;
  a.D = c->D;
  a.C = c->C;
  a.nf = nf;
  a.nt = nt;
  a.pre_mode = pre;
  a.post_mode = post;
  a.out_scale = out_scale;
  const int nmax = std::max(nf, nt);
  const int cap = c->D == 3 ? nmax * nmax * nmax : nmax * nmax;
  const size_t smem = sizeof(double) * (2 * (size_t)c->C * cap + nt * nf);
  ensure_smem(sweep_all_kernel, smem);
  if (c->E == 0) return;
  sweep_all_kernel<<<(unsigned)c->E, 256, smem, s>>>(a);
  WK_CUDA(cudaGetLastError());
}

TckProgram& get_program(wk_ctx* c, int policy, int shift) {
  const int key = policy * 2 + (shift ? 1 : 0);
  const bool gl_full = c->mode == WK_GEOM_AFFINE;  // full degree in GL (affine) or Gauss
  auto it = c->progs.find(key);
  if (it != c->progs.end()) return it->second;
  const int k = c->k, D = c->D;
  std::vector<int> ops;
  std::vector<double> wts;  // filled with Taylor index j; weights set per call
  std::vector<long double> tab;
  std::map<int, int> slot;  // degree -> offset
  int acc_len = 0;
  auto npts = [&](int q) { int n = q + 1; return D == 3 ? n * n * n : n * n; };
  auto add_tab = [&](const Mat& m) {
    int off = (int)tab.size();
    tab.insert(tab.end(), m.begin(), m.end());
    return off;
  };
  auto alloc_slot = [&](int q) {
    slot[q] = acc_len;
    acc_len += (D + 1) * npts(q);
  };
  auto emit = [&](int code, int a0, int a1, int a2, double w) {
    ops.insert(ops.end(), {code, a0, a1, a2});
    wts.push_back(w);
  };
  // resize matrix from degree a to b with the full degree in the GL basis
  auto resize_mat = [&](int a, int b) {
    if (!gl_full) return resize_gauss(a, b);
    if (a == k) {  // GL(k) -> Gauss(b): P_{k->b} B_k
      return matmul(resize_gauss(k, b), table_B(k), b + 1, k + 1, k + 1);
    }
    if (b == k) return lagrange(g_nodes(a), gl_nodes(k), false);  // Gauss(a) -> GL(k)
    return resize_gauss(a, b);
  };
  alloc_slot(k);
  emit(TCK_ACC_SET, slot[k], k + 1, 0, shift ? -2.0 : -1.0);  // weight index encoded
  auto sched = schedule(k, policy);
  const int n_apps = shift ? std::max(k - 1, 0) : k + 1;
  int deg = k;
  for (int j = 1; j <= n_apps; ++j) {
    const int din = sched[j - 1].first, dout = sched[j - 1].second;
    if (din == 0) break;
    emit(TCK_S, deg + 1, add_tab(deg == k && gl_full ? table_Dglco(k) : table_Dco(deg)), 0, 0.0);
    if (dout != din) {
      emit(TCK_RESIZE, deg + 1, dout + 1, add_tab(resize_mat(deg, dout)), 0.0);
      deg = dout;
    }
    const int widx = shift ? j + 1 : j;
    if (slot.count(deg)) {
      emit(TCK_ACC_ADD, slot[deg], deg + 1, 0, -1.0 - widx);
    } else {
      alloc_slot(deg);
      emit(TCK_ACC_SET, slot[deg], deg + 1, 0, -1.0 - widx);
    }
  }
  for (auto itl = slot.begin(); itl != slot.end(); ++itl) {
    const int lo = itl->first;
    if (lo == k) break;
    auto ith = std::next(itl);
    const int hi = ith->first;
    emit(TCK_LOAD, slot[lo], lo + 1, 0, 0.0);
    emit(TCK_RESIZE, lo + 1, hi + 1, add_tab(resize_mat(lo, hi)), 0.0);
    emit(TCK_ACC_ADD, slot[hi], hi + 1, 0, 1.0);
  }
  TckProgram p;
  p.nops = (int)wts.size();
  p.acc_len = acc_len;
  p.tab_len = (int)tab.size();
  p.d_ops = upload(ops.data(), ops.size());
  auto tabd = std::vector<double>(tab.begin(), tab.end());
  p.d_tab = upload(tabd.data(), tabd.size());
  p.h_ops = ops;
  p.h_tab = tabd;
  // weights: negative entries encode Taylor indices -(1+j); resolved per dt
  p.enc = wts;
  c->progs[key] = p;
  return c->progs[key];
}

// The Taylor weights of a program for a given dt (resolved on the host and
// passed by value in the launch arguments: no device buffer, no sync).
double program_weight(const TckProgram& p, int i, double dt) {
  return p.enc[i] < 0.0 ? taylor_weight((int)(-p.enc[i] - 1.0 + 0.5), dt) : p.enc[i];
}

void run_ader_a(wk_ctx* c, bool hdg, const double* U, double* V, double* Y, double dt,
                int policy, int shift, cudaStream_t s, int y_mode = 0) {
  TckProgram& p = get_program(c, policy, shift);
  auto plan_check = [&]() {
    // compile-time plan: valid when it reproduces this program op for op
    if (p.plan_ok < 0) {
      const TckPlan pl = make_tck_plan(c->k, reduction_stride(policy), shift != 0);
      bool ok = pl.n == p.nops && pl.tab_len == (int)p.h_tab.size() && pl.n <= kPlanOps &&
                pl.tab_len <= kPlanTab;
      for (int i = 0; ok && i < pl.n; ++i) {
        const int* o = &p.h_ops[4 * i];
        const TckStep& q = pl.ops[i];
        ok = o[0] == q.code &&
             (q.code == TCK_S ? (o[1] == q.a0 && o[2] == q.a1)
              : q.code == TCK_RESIZE ? (o[1] == q.a0 && o[2] == q.a1 && o[3] == q.a2)
                                      : o[2] == q.a1);
      }
      p.plan_ok = ok ? 1 : 0;
    }
    return p.plan_ok == 1;
  };
  auto stream_tck_args = [&]() {
    TckStreamArgs sa{};
    sa.op = affine_args(c);
    sa.op.u = U;
    sa.y = Y;
    sa.v_out = V;
    sa.dt = dt;
    for (int i = 0; i < p.nops; ++i) sa.w[i] = program_weight(p, i, dt);
    for (size_t i = 0; i < p.h_tab.size(); ++i) sa.tab[i] = p.h_tab[i];
    return sa;
  };
  if (c->mode == WK_GEOM_CURVED && y_mode == 0 && stream_curved_supported(c->D, c->N) &&
      stream_ader_enabled() && plan_check()) {
    CurvedStreamArgs ca = curved_stream_args(c);
    ca.t = stream_tck_args();
    bool done = false;
    dispatch_dn<CurvedStream>(c->D, c->N, hdg ? kCurvedAderHdg : kCurvedAder,
                              reduction_stride(policy), shift != 0, ca, s, done);
    if (done) return;
  }
  if (c->mode == WK_GEOM_AFFINE && c->cart && c->d_cls == nullptr &&
      stream_ader_supported(c->D, c->N) && stream_ader_enabled()) {
    if (plan_check()) {
      const TckStreamArgs sa = stream_tck_args();
      bool done = false;
      dispatch_dn<StreamAderA>(c->D, c->N, hdg, reduction_stride(policy), shift != 0, sa, s,
                               done);
      if (done) return;
    }
  }
  TckArgs a{};
  a.op = affine_args(c);
  a.op.u = U;
  a.y = Y;
  a.v_out = V;
  a.prog = p.d_ops;
  require(p.nops <= kTckOps, "TCK program too long");
  for (int i = 0; i < p.nops; ++i) a.w[i] = program_weight(p, i, dt);
  a.tck_tab = p.d_tab;
  a.nops = p.nops;
  a.tab_len = p.tab_len;
  a.acc_len = p.acc_len;
  a.dt = dt;
  if (c->mode == WK_GEOM_AFFINE) {
    const bool fast = c->cart && c->d_cls == nullptr;  // warp-group kernel handles HDG fused
    if (hdg && !fast) {
      // general affine ADER-HDG: W = M^{-1} K U into Y (stage kernel), V = U - dt W,
      // then the Taylor loop on W in place (Y -> y); DESIGN.md §8.
      AffineArgs o = affine_args(c);
      o.u = U;
      o.out = Y;
      run_op(c, OUT_MINVK, o, s);
      const long long n = (long long)c->rcount() * c->C * c->NODES;
      const long long off = (long long)c->rbegin() * c->C * c->NODES;
      if (n > 0) {
        axpy_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 32), 256, 0, s>>>(
            U + off, Y + off, V + off, dt, n);
        WK_CUDA_AT(cudaGetLastError(), "axpy_kernel");
      }
      a.op.u = Y;
      dispatch_dn<AderA>(c->D, c->N, c, false, a, s);
      return;
    }
    dispatch_dn<AderA>(c->D, c->N, c, hdg, a, s);
  } else {
    CurvedArgs g = curved_args(c);
    g.y_mode = y_mode;
    dispatch_dn<CurvedAderA>(c->D, c->N, hdg, a, g, s);
  }
}

template <int D, int N>
struct SmallRun {
  static void run(const SmallArgs& a, cudaStream_t s, bool dry, bool& ok) {
    ok = small_lsrk_launch<D, N>(a, s, dry);
  }
};

// the whole-run cluster kernel covers Cartesian single-class affine meshes
// without halo slots, launched over the full element range
bool small_eligible(const wk_ctx* c) {
  return c->mode == WK_GEOM_AFFINE && c->cart && c->d_cls == nullptr && c->G == 0 &&
         c->range_count < 0 && c->E > 0;
}

SmallArgs small_args(wk_ctx* c) {
  SmallArgs a{};
  a.nbr = c->d_nbr;
  a.mat = c->d_mat;
  a.geo = c->d_geo;
  a.E = c->E;
  a.stab = c->stab;
  const int n = c->N;
  for (int i = 0; i < n * n; ++i) a.cA[i] = c->h_optab[i];
  for (int i = 0; i < n; ++i) {
    a.cL0[i] = c->h_optab[n * n + i];
    a.cL1[i] = c->h_optab[n * n + n + i];
  }
  return a;
}

// One export face per blockIdx.y row, its C x NF values over the x
// threads: 32-bit index arithmetic (the flat version did three 64-bit
// divisions per value).  send[i] = the (C, NF) face slice of export i.
__global__ void pack_halo_kernel(const double* u, double* send, const long long* elem,
                                 const int* face, long long n, int C, int N, int D) {
  const int NF = D == 3 ? N * N : N;
  const int NODES = D == 3 ? N * N * N : N * N;
  const int per = C * NF;
  const int t = threadIdx.x;
  if (t >= per) return;
  const int c = t / NF, fn = t - c * NF;
  for (long long i = blockIdx.x; i < n; i += gridDim.x) {
    const int f = face[i];
    const int m = f >> 1, sd = f & 1;
    const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
    const int node = fn % sm + sd * (N - 1) * sm + (fn / sm) * sm * N;
    send[i * per + t] = u[(elem[i] * C + c) * NODES + node];
  }
}

}  // namespace

// ===========================================================================
extern "C" {

int wk_version(void) { return 1; }
const char* wk_last_error(void) { return g_err.c_str(); }

int wk_ctx_create(const wk_desc* desc, wk_ctx** out) {
  return guarded([&] {
    require(desc && out, "null argument");
    require(desc->dim == 2 || desc->dim == 3, "dimension must be 2 or 3");
    require(desc->degree >= 1 && desc->degree <= kMaxN - 1, "degree must be in 1..8");
    require(desc->n_elements >= 0, "negative element count");
    auto* c = new wk_ctx();
    try {
      c->D = desc->dim;
      c->k = desc->degree;
      c->N = c->k + 1;
      c->C = c->D + 1;
      c->NODES = c->D == 3 ? c->N * c->N * c->N : c->N * c->N;
      c->NF = c->D == 3 ? c->N * c->N : c->N;
      c->E = desc->n_elements;
      c->G = desc->n_ghost_faces;
      c->stab = desc->stabilization ? 1 : 0;
      c->mode = desc->geometry_mode;
      const long long E = c->E;
      const int D = c->D;
      require(c->G >= 0, "negative ghost face count");
      // every neighbour code must name an element, the wall (-1) or a ghost
      // slot of the halo buffer: the kernels gather through them unchecked
      for (long long i = 0; i < E * 2 * D; ++i) {
        const int v = desc->neighbors[i];
        require(v < E && (v >= -1 || (long long)(-2 - v) < c->G),
                "neighbour table entry out of range (element, -1 wall or ghost slot)");
      }
      c->d_nbr = upload(desc->neighbors, (size_t)E * 2 * D);
      WK_CUDA(cudaMalloc(&c->d_sched, 4 * sizeof(unsigned)));
      WK_CUDA(cudaMemset(c->d_sched, 0, 4 * sizeof(unsigned)));
      std::vector<double> mat((size_t)E * kMatStride, 0.0);
      for (long long e = 0; e < E; ++e) {
        require(desc->tau[e] > 0.0, "stabilization must be positive");
        mat[e * kMatStride + 0] = desc->inv_rho[e];
        mat[e * kMatStride + 1] = desc->c2rho[e];
        mat[e * kMatStride + 2] = desc->tau[e];
        mat[e * kMatStride + 3] = desc->inv_rho[e] / desc->tau[e];  // ir/tau, no device division
      }
      c->d_mat = upload(mat.data(), mat.size());
      if (c->G > 0)
        WK_CUDA(cudaMalloc(&c->d_ghost, sizeof(double) * (size_t)c->G * c->C * c->NF));
      auto A = to_double(table_A(c->k)), L = to_double(table_lift(c->k));
      std::vector<double> optab(A);
      optab.insert(optab.end(), L.begin(), L.end());
      c->d_optab = upload(optab.data(), optab.size());
      c->h_optab = optab;
      if (c->mode == WK_GEOM_AFFINE) {
        const long long nc = desc->n_classes;
        require(nc >= 1, "affine geometry needs at least one class");
        require(nc == 1 || desc->geo_class, "geo_class required for n_classes > 1");
        c->n_classes = nc;
        const int st = D == 3 ? GeoLayout<3>::STRIDE : GeoLayout<2>::STRIDE;
        std::vector<double> geo((size_t)nc * st, 0.0);
        bool cart = true;
        for (long long q = 0; q < nc; ++q) {
          double* g = geo.data() + q * st;
          for (int i = 0; i < D * D; ++i) {
            g[i] = desc->affine_G[q * D * D + i];
            if (i / D != i % D && g[i] != 0.0) cart = false;
          }
          for (int i = 0; i < 2 * D * D; ++i) g[D * D + i] = desc->affine_normal[q * 2 * D * D + i];
          for (int i = 0; i < 2 * D; ++i) g[3 * D * D + i] = desc->affine_fscale[q * 2 * D + i];
          g[3 * D * D + 2 * D] = desc->affine_det[q];
          require(desc->affine_det[q] > 0.0, "non-positive Jacobian determinant");
        }
        c->cart = cart ? 1 : 0;
        c->d_geo = upload(geo.data(), geo.size());
        if (desc->geo_class) {
          for (long long e = 0; e < E; ++e)
            require(desc->geo_class[e] >= 0 && desc->geo_class[e] < nc, "geo_class out of range");
          c->d_cls = upload(desc->geo_class, (size_t)E);
        }
      } else if (c->mode == WK_GEOM_CURVED) {
        curved_setup(c, desc);
      } else {
        throw WkError(WK_EINVAL, "unknown geometry mode");
      }
      *out = c;
    } catch (...) {
      wk_ctx_destroy(c);
      throw;
    }
  });
}

int wk_ctx_destroy(wk_ctx* c) {
  if (!c) return WK_OK;
  cudaFree(c->d_nbr);
  cudaFree(c->d_sched);
  cudaFree(c->d_mat);
  cudaFree(c->d_geo);
  cudaFree(c->d_cls);
  if (c->own_ghost) cudaFree(c->d_ghost);
  cudaFree(c->d_optab);
  cudaFree(c->scratch);
  cudaFree(c->d_exp_elem);
  cudaFree(c->d_exp_face);
  for (auto& kv : c->tables) cudaFree(kv.second);
  for (auto& kv : c->progs) {
    cudaFree(kv.second.d_ops);
    cudaFree(kv.second.d_tab);
  }
  for (double* p : c->owned) cudaFree(p);
  delete c;
  return WK_OK;
}

int wk_apply_minv_K(wk_ctx* c, const double* u, double* out, int parts, void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(parts >= 1 && parts <= 3, "parts must be cell, face or both");
    require(u != out, "input and output must not alias");
    AffineArgs a = affine_args(c);
    a.u = u;
    a.out = out;
    a.parts = parts;
    run_op(c, OUT_MINVK, a, (cudaStream_t)stream);
  });
}

int wk_rhs(wk_ctx* c, const double* u, double* out, void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(u != out, "input and output must not alias");
    AffineArgs a = affine_args(c);
    a.u = u;
    a.out = out;
    run_op(c, OUT_RHS, a, (cudaStream_t)stream);
  });
}

int wk_apply_mass(wk_ctx* c, const double* x, double* y, void* stream);

int wk_apply_K(wk_ctx* c, const double* u, double* out, int parts, void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(parts >= 1 && parts <= 3, "parts must be cell, face or both");
    require(u != out, "input and output must not alias");
    if (c->mode == WK_GEOM_CURVED) {
      AffineArgs a = affine_args(c);
      a.u = u;
      a.out = out;
      a.parts = parts;
      dispatch_dn<CurvedOp>(c->D, c->N, (int)OUT_K, a, curved_args(c), (cudaStream_t)stream);
      return;
    }
    // K u = M (M^{-1} K u)  -- exact on affine cells
    double* tmp = c->scratch_buf();
    AffineArgs a = affine_args(c);
    a.u = u;
    a.out = tmp;
    a.parts = parts;
    run_op(c, OUT_MINVK, a, (cudaStream_t)stream);
    sweep(c, tmp, out, c->table("M1", table_M1(c->k)), c->N, c->N, SCALE_NONE, SCALE_DET,
          nullptr, 1.0, (cudaStream_t)stream);
  });
}

int wk_apply_inverse_mass(wk_ctx* c, const double* x, double* y, void* stream) {
  return guarded([&] {
    require(c, "null context");
    cudaStream_t s = (cudaStream_t)stream;
    if (c->mode == WK_GEOM_AFFINE) {
      sweep(c, x, y, c->table("M1inv", inverse(table_M1(c->k), c->N)), c->N, c->N, SCALE_NONE,
            SCALE_INV_DET, nullptr, 1.0, s);
    } else {
      require(x != y, "input and output must not alias");
      // B^{-1} [ (B^{-T} x) / JxW ]   (operator.py:250-258)
      const Mat binv = table_Binv(c->k);
      double* tmp = c->scratch_buf();
      sweep(c, x, tmp, c->table("BinvT", transpose(binv, c->N, c->N)), c->N, c->N, SCALE_NONE,
            SCALE_NONE, nullptr, 1.0, s);
      sweep(c, tmp, y, c->table("Binv", binv), c->N, c->N, SCALE_DIV_PTS, SCALE_NONE,
            c->d_jxw.at(c->k), 1.0, s);
    }
  });
}

// Mass-weighted squared norm u . M u = sum_e sum_q JxW_q (B u)_q^2, fused
// (state_norm, stepping.py:321-324: sqrt(|vdot(u, M u)|)); per-element
// partials reduced in a fixed order, result left on the device.
int wk_state_norm_sq(wk_ctx* c, const double* u, double* out_sq, void* stream) {
  return guarded([&] {
    require(c, "null context");
    cudaStream_t s = (cudaStream_t)stream;
    const long long E = c->E;
    if (E == 0) {
      WK_CUDA(cudaMemsetAsync(out_sq, 0, sizeof(double), s));
      return;
    }
    const int n = c->N, D = c->D, C = D + 1, nodes = c->NODES;
    std::vector<long double> gp, gw;
    gauss_rule(n, gp, gw);
    const double* B = c->table("B", table_B(c->k));
    const double* w = c->table("GW", Mat(gw.begin(), gw.end()));
    const double* jxw = c->mode == WK_GEOM_CURVED ? c->d_jxw.at(c->k) : nullptr;
    const size_t smem = sizeof(double) * (2 * C * nodes + n * n + fields::kThreads);
    double* part = c->part_buf();
    if (D == 3) {
      ensure_smem(fields::mass_norm_kernel<3>, smem);
      fields::mass_norm_kernel<3><<<(unsigned)E, fields::kThreads, smem, s>>>(
          u, n, B, w, jxw, c->d_geo, GeoLayout<3>::STRIDE, GeoLayout<3>::DET, c->d_cls, part);
    } else {
      ensure_smem(fields::mass_norm_kernel<2>, smem);
      fields::mass_norm_kernel<2><<<(unsigned)E, fields::kThreads, smem, s>>>(
          u, n, B, w, jxw, c->d_geo, GeoLayout<2>::STRIDE, GeoLayout<2>::DET, c->d_cls, part);
    }
    WK_CUDA_AT(cudaGetLastError(), "mass_norm_kernel");
    fields::ordered_sum_kernel<<<1, fields::kThreads, 0, s>>>(part, E, out_sq);
    WK_CUDA_AT(cudaGetLastError(), "ordered_sum_kernel");
  });
}

int wk_apply_mass(wk_ctx* c, const double* x, double* y, void* stream) {
  return guarded([&] {
    require(c, "null context");
    cudaStream_t s = (cudaStream_t)stream;
    if (c->mode == WK_GEOM_AFFINE) {
      sweep(c, x, y, c->table("M1", table_M1(c->k)), c->N, c->N, SCALE_NONE, SCALE_DET, nullptr,
            1.0, s);
    } else {
      require(x != y, "input and output must not alias");
      const Mat b = table_B(c->k);
      double* tmp = c->scratch_buf();
      sweep(c, x, tmp, c->table("B", b), c->N, c->N, SCALE_NONE, SCALE_MUL_PTS,
            c->d_jxw.at(c->k), 1.0, s);
      sweep(c, tmp, y, c->table("BT", transpose(b, c->N, c->N)), c->N, c->N, SCALE_NONE,
            SCALE_NONE, nullptr, 1.0, s);
    }
  });
}

int wk_to_gauss_values(wk_ctx* c, const double* x, double* y, void* stream) {
  return guarded([&] {
    require(c, "null context");
    sweep(c, x, y, c->table("B", table_B(c->k)), c->N, c->N, SCALE_NONE, SCALE_NONE, nullptr, 1.0,
          (cudaStream_t)stream);
  });
}

int wk_from_gauss_weighted(wk_ctx* c, const double* x, double* y, void* stream) {
  return guarded([&] {
    require(c, "null context");
    cudaStream_t s = (cudaStream_t)stream;
    if (c->mode == WK_GEOM_AFFINE) {
      // B^T (JxW x) with JxW = det * (w x w x w)
      sweep(c, x, y, c->table("BtW", table_BtW(c->k)), c->N, c->N, SCALE_NONE, SCALE_DET,
            nullptr, 1.0, s);
    } else {
      const Mat b = table_B(c->k);
      sweep(c, x, y, c->table("BT", transpose(b, c->N, c->N)), c->N, c->N, SCALE_MUL_PTS,
            SCALE_NONE, c->d_jxw.at(c->k), 1.0, s);
    }
  });
}

int wk_apply_local_S(wk_ctx* c, const double* x, double* y, int degree, void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(degree >= 0 && degree <= c->k, "degree outside 0..k");
    require(x != y, "input and output must not alias");
    LocalSArgs a{};
    a.in = x;
    a.out = y;
    a.dco = c->table("Dco" + std::to_string(degree), table_Dco(degree));
    a.mat = c->d_mat;
    a.E = c->E;
    a.D = c->D;
    a.nq = degree + 1;
    if (c->mode == WK_GEOM_AFFINE) {
      a.geo = c->d_geo;
      a.geo_class = c->d_cls;
      a.geo_stride = c->D == 3 ? GeoLayout<3>::STRIDE : GeoLayout<2>::STRIDE;
    } else {
      auto it = c->d_invjac.find(degree);
      require(it != c->d_invjac.end(),
              "geometry has no degree-" + std::to_string(degree) + " point set");
      a.inv_jac = it->second;
    }
    const int np = c->D == 3 ? a.nq * a.nq * a.nq : a.nq * a.nq;
    const size_t smem = sizeof(double) * ((size_t)c->C * np + a.nq * a.nq);
    ensure_smem(local_S_kernel, smem);
    if (c->E == 0) return;
    local_S_kernel<<<(unsigned)c->E, 256, smem, (cudaStream_t)stream>>>(a);
    WK_CUDA(cudaGetLastError());
  });
}

int wk_resize_values(wk_ctx* c, const double* x, double* y, int k_from, int k_to,
                     void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(k_from >= 0 && k_to >= 0 && k_from <= kMaxN - 1 && k_to <= kMaxN - 1,
            "degree out of range");
    require(x != y, "input and output must not alias");
    const std::string key = "R" + std::to_string(k_from) + "_" + std::to_string(k_to);
    sweep(c, x, y, c->table(key, resize_gauss(k_from, k_to)), k_from + 1, k_to + 1, SCALE_NONE,
          SCALE_NONE, nullptr, 1.0, (cudaStream_t)stream);
  });
}

int wk_lsrk_stage_ex(wk_ctx* c, const double* u_in, double* u_out, double* r, double a_,
                     double b_, double dt, int r_dead, void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(u_in != u_out, "u_out must not alias u_in");
    AffineArgs a = affine_args(c);
    a.u = u_in;
    a.u_out = u_out;
    a.r = r;
    a.a = a_;
    a.b = b_;
    a.dt = dt;
    a.r_dead = r_dead != 0;
    run_op(c, OUT_LSRK, a, (cudaStream_t)stream);
  });
}

int wk_lsrk_stage(wk_ctx* c, const double* u_in, double* u_out, double* r, double a_,
                  double b_, double dt, void* stream) {
  return wk_lsrk_stage_ex(c, u_in, u_out, r, a_, b_, dt, 0, stream);
}

int wk_lsrk_run_supported(wk_ctx* c) {
  if (!c || !small_eligible(c)) return 0;
  try {
    bool ok = false;
    dispatch_dn<SmallRun>(c->D, c->N, small_args(c), (cudaStream_t)0, true, ok);
    return ok ? 1 : 0;
  } catch (...) {
    return 0;
  }
}

int wk_lsrk_run(wk_ctx* c, const double* u_in, double* u_out, int n_stages, const double* a_,
                const double* b_, double dt, int n_steps, void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(small_eligible(c), "mesh not eligible for the whole-run cluster kernel "
                               "(Cartesian single-class affine, no halo, small enough)");
    require(n_stages >= 1 && n_stages <= kSmallMaxStages && n_steps >= 0, "bad stage / step count");
    require(a_[0] == 0.0, "the first LSRK stage must have a = 0");
    SmallArgs a = small_args(c);
    a.u_in = u_in;
    a.u_out = u_out;
    a.stages = n_stages;
    a.steps = n_steps;
    a.dt = dt;
    for (int i = 0; i < n_stages; ++i) {
      a.a[i] = a_[i];
      a.b[i] = b_[i];
    }
    bool ok = false;
    dispatch_dn<SmallRun>(c->D, c->N, a, (cudaStream_t)stream, false, ok);
    require(ok, "mesh too large for the whole-run cluster kernel");
  });
}

int wk_tck(wk_ctx* c, const double* w, double* t_out, double dt, int policy, int shift,
           void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(w != t_out, "input and output must not alias");
    // reference returns the mass-weighted T = B^T (JxW acc_k)  (stepping.py:261)
    if (c->mode == WK_GEOM_AFFINE) {
      double* y = c->scratch_buf();
      run_ader_a(c, false, w, nullptr, y, dt, policy, shift, (cudaStream_t)stream);
      sweep(c, y, t_out, c->table("M1", table_M1(c->k)), c->N, c->N, SCALE_NONE, SCALE_DET,
            nullptr, 1.0, (cudaStream_t)stream);
    } else {
      run_ader_a(c, false, w, nullptr, t_out, dt, policy, shift, (cudaStream_t)stream, 1);
    }
  });
}

int wk_ader_a(wk_ctx* c, int variant, int policy, const double* U, double* V, double* Y,
              double dt, void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(variant == WK_ADER || variant == WK_ADER_HDG, "unknown ader variant");
    require(U && Y && U != Y, "ADER needs distinct U and Y buffers");
    require(variant == WK_ADER || (V && V != U && V != Y), "ADER-HDG needs a distinct V buffer");
    const bool hdg = variant == WK_ADER_HDG;
    run_ader_a(c, hdg, U, V, Y, dt, policy, hdg ? 1 : 0, (cudaStream_t)stream);
  });
}

int wk_ader_b(wk_ctx* c, int variant, double* U, const double* V, const double* Y,
              void* stream) {
  return guarded([&] {
    require(c, "null context");
    require(variant == WK_ADER || variant == WK_ADER_HDG, "unknown ader variant");
    require(U && Y && U != Y, "ADER needs distinct U and Y buffers");
    AffineArgs a = affine_args(c);
    a.u = Y;
    a.v = variant == WK_ADER_HDG ? V : U;
    a.out = U;
    run_op(c, OUT_ADERB, a, (cudaStream_t)stream);
  });
}

int wk_ader_step(wk_ctx* c, int variant, int policy, double* U, double* V, double* Y, double dt,
                 void* stream) {
  const int rc = wk_ader_a(c, variant, policy, U, V, Y, dt, stream);
  if (rc != WK_OK) return rc;
  return wk_ader_b(c, variant, U, V, Y, stream);
}

double* wk_ghost_buffer(wk_ctx* c) { return c ? c->d_ghost : nullptr; }

int wk_set_ghost_buffer(wk_ctx* c, double* ghost) {
  return guarded([&] {
    require(c && ghost, "null argument");
    require(c->G > 0, "context was created without ghost face slots");
    if (c->own_ghost) cudaFree(c->d_ghost);
    c->d_ghost = ghost;
    c->own_ghost = false;
  });
}

int wk_set_halo_exports(wk_ctx* c, int64_t n, const int64_t* elem, const int32_t* face) {
  return guarded([&] {
    require(c && n >= 0, "bad arguments");
    cudaFree(c->d_exp_elem);
    cudaFree(c->d_exp_face);
    c->d_exp_elem = nullptr;
    c->d_exp_face = nullptr;
    c->n_export = n;
    for (int64_t i = 0; i < n; ++i) {
      require(elem[i] >= 0 && elem[i] < c->E, "export element out of range");
      require(face[i] >= 0 && face[i] < 2 * c->D, "export face out of range");
    }
    c->d_exp_elem = upload(reinterpret_cast<const long long*>(elem), (size_t)n);
    c->d_exp_face = upload(face, (size_t)n);
  });
}

int wk_pack_halo(wk_ctx* c, const double* u, double* send, void* stream) {
  return guarded([&] {
    require(c, "null context");
    if (c->n_export == 0) return;
    const int threads = (c->C * c->NF + 31) / 32 * 32;   // <= 4 * 81 -> 352
    const int blocks = (int)std::min<long long>(c->n_export, 148 * 16);
    pack_halo_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
        u, send, c->d_exp_elem, c->d_exp_face, c->n_export, c->C, c->N, c->D);
    WK_CUDA(cudaGetLastError());
  });
}

int wk_set_element_range(wk_ctx* c, int64_t begin, int64_t count) {
  return guarded([&] {
    require(c, "null context");
    if (count < 0) {
      c->range_begin = 0;
      c->range_count = -1;
      return;
    }
    require(begin >= 0 && begin + count <= c->E, "element range out of bounds");
    c->range_begin = begin;
    c->range_count = count;
  });
}

int wk_debug_set_neighbor(wk_ctx* c, int64_t element, int face, int32_t value) {
  return guarded([&] {
    require(c && element >= 0 && element < c->E && face >= 0 && face < 2 * c->D,
            "bad element / face");
    WK_CUDA(cudaMemcpy(c->d_nbr + element * 2 * c->D + face, &value, sizeof(int32_t),
                       cudaMemcpyHostToDevice));
  });
}

int wk_set_tile_order(wk_ctx* c, int64_t chunk, int64_t n_slow, int64_t n_blocks) {
  return guarded([&] {
    require(c, "null context");
    if (chunk <= 0) {
      c->tord_ch = c->tord_ns = c->tord_nb = 0;
      return;
    }
    require(n_slow > 0 && n_blocks > 0 && chunk * n_slow * n_blocks == c->E,
            "tile order must cover the element range exactly");
    require(c->E < (1LL << 32), "tile order needs fewer than 2^32 elements");
    c->tord_ch = chunk;
    c->tord_ns = n_slow;
    c->tord_nb = n_blocks;
  });
}

int wk_set_queue_slot(wk_ctx* c, int slot) {
  return guarded([&] {
    require(c, "null context");
    require(slot == 0 || slot == 1, "queue slot must be 0 or 1");
    c->queue_slot = slot;
  });
}

int wk_basis_table(int kind, int k, int k_to, double* out, int out_len) {
  try {
    if (k < 0 || k > 12) return -1;
    std::vector<long double> v;
    std::vector<long double> x, w;
    switch (kind) {
      case WK_TABLE_GAUSS_POINTS: gauss_rule(k + 1, x, w); v = x; break;
      case WK_TABLE_GAUSS_WEIGHTS: gauss_rule(k + 1, x, w); v = w; break;
      case WK_TABLE_GL_POINTS:
        if (k == 0) return -1;
        gauss_lobatto_rule(k + 1, x, w); v = x; break;
      case WK_TABLE_GL_WEIGHTS:
        if (k == 0) return -1;
        gauss_lobatto_rule(k + 1, x, w); v = w; break;
      case WK_TABLE_GL_TO_G: v = table_B(k); break;
      case WK_TABLE_G_TO_GL: v = table_Binv(k); break;
      case WK_TABLE_D_GL: v = table_Dgl(k); break;
      case WK_TABLE_D_CO: v = table_Dco(k); break;
      case WK_TABLE_RESIZE:
        if (k_to < 0 || k_to > 12) return -1;
        v = resize_gauss(k, k_to); break;
      case WK_TABLE_A_SPLIT: if (k == 0) return -1; v = table_A(k); break;
      case WK_TABLE_LIFT: if (k == 0) return -1; v = table_lift(k); break;
      default: return -1;
    }
    if ((int)v.size() > out_len) return -1;
    for (size_t i = 0; i < v.size(); ++i) out[i] = (double)v[i];
    return (int)v.size();
  } catch (...) {
    return -1;
  }
}

}  // extern "C"

namespace wk {
void set_last_error(const char* msg) { g_err = msg; }
}  // namespace wk
