/*
 * wavekernel_b200 — C ABI of the B200-native DG-acoustics hot path.
 *
 * Drop-in boundary for the reference package `wavekernel`
 * (/root/reference/pkg/src/wavekernel).  The reference has no FFI of its own:
 * its steppers reach the operator through duck-typed Python method calls
 * (SURVEY.md §8b).  Each entry point below replaces one of those methods or
 * one fused composition of them; the reference interface it replaces is cited
 * beside it.  The Python mirror (paper_1805_03981_b200/operator.py,
 * stepping.py) binds these through ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Every function returns 0 on success and a nonzero WK_E* code on failure;
 *    wk_last_error() returns a thread-local message for the last failure
 *    (the Python layer raises ValueError / RuntimeError from it, like the
 *    reference's ValueError checks in operator.py:96-133, :288-290).
 *  - State pointers are DEVICE pointers owned by the caller, FP64, layout
 *    (E, d+1, n, ..., n) element-contiguous, components v_1..v_d, p,
 *    direction 0 fastest (reference StateVector, operator.py:33-55).
 *    Inputs and outputs must not alias unless stated.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); every call is
 *    asynchronous on it.
 *  - Host arrays in wk_desc are copied into context-owned device memory by
 *    wk_ctx_create; the caller may free them afterwards.
 */
#ifndef WAVEKERNEL_B200_H
#define WAVEKERNEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WK_OK 0
#define WK_EINVAL 1     /* bad argument / unsupported configuration */
#define WK_ECUDA 2      /* CUDA runtime error */
#define WK_ESTATE 3     /* context not ready for this call */

#define WK_GEOM_AFFINE 0  /* per-element constant Jacobian (multilinear = affine cells) */
#define WK_GEOM_CURVED 1  /* per-point metric arrays (reference GeometryCache layout) */

#define WK_PART_CELL 1    /* apply_K(parts="cell")  operator.py:157 */
#define WK_PART_FACE 2    /* apply_K(parts="face")  operator.py:189 */
#define WK_PART_BOTH 3

#define WK_POLICY_NONE 0          /* kernels.py REDUCTION_STRIDE */
#define WK_POLICY_EVERY_STEP 1
#define WK_POLICY_EVERY_SECOND 2
#define WK_POLICY_EVERY_THIRD 3

#define WK_ADER 0       /* ader_step(variant="ader")      stepping.py:271-276 */
#define WK_ADER_HDG 1   /* ader_step(variant="ader_hdg")  stepping.py:277-284 */

typedef struct wk_ctx wk_ctx;

/* Operator description: mirrors AcousticOperator(mesh, geometry, material,
 * flux) (operator.py:93-123).  Neighbour codes: >=0 local element, -1
 * sound-soft wall (operator.py:217-220), <= -2 ghost face slot (-2-g) of the
 * halo buffer (multi-GPU slabs). */
typedef struct wk_desc {
  int32_t dim;                 /* d in {2,3} */
  int32_t degree;              /* k in 1..8 */
  int64_t n_elements;          /* E (local elements) */
  int64_t n_ghost_faces;       /* G, halo face slots (0 on one GPU) */
  const int32_t* neighbors;    /* (E, d, 2)  Mesh.neighbors, mesh.py:96-107 */
  const double* inv_rho;       /* (E,)  1/rho            operator.py:116 */
  const double* c2rho;         /* (E,)  c^2 rho          operator.py:117 */
  const double* tau;           /* (E,)  HDG tau          operator.py:118-123 */
  int32_t stabilization;       /* FluxParams.stabilization operator.py:58-67 */
  int32_t geometry_mode;       /* WK_GEOM_* */
  /* WK_GEOM_AFFINE: per-class constants; element e uses class geo_class[e]
   * (geo_class may be NULL when n_classes == 1). */
  int64_t n_classes;
  const int32_t* geo_class;    /* (E,) */
  const double* affine_G;      /* (n_classes, d, d)   d xi_m / d x_i  (inv_jac) */
  const double* affine_det;    /* (n_classes,)        det J          */
  const double* affine_normal; /* (n_classes, d, 2, d) outward unit normal of face (m,s) */
  const double* affine_fscale; /* (n_classes, d, 2)   face JxW / (w x w) / det J */
  /* WK_GEOM_CURVED: reference GeometryCache arrays (mesh.py:162-188).
   * vol arrays for each degree in curved_degrees (first = k). */
  int32_t n_curved_degrees;
  const int32_t* curved_degrees;       /* (n_curved_degrees,) */
  const double* const* curved_inv_jac; /* per degree q: (E, d, d, (q+1)^d) */
  const double* const* curved_jxw;     /* per degree q: (E, (q+1)^d) */
  const double* const* face_normal;    /* per face 2m+s: (E, d, (k+1)^(d-1)) */
  const double* const* face_jxw;       /* per face 2m+s: (E, (k+1)^(d-1)) */
} wk_desc;

int wk_version(void);
const char* wk_last_error(void);

int wk_ctx_create(const wk_desc* desc, wk_ctx** out);
int wk_ctx_destroy(wk_ctx* ctx);

/* ---- operator calls (AcousticOperator methods) ---------------------- */
/* apply_K(state, parts)                         operator.py:149-191 */
int wk_apply_K(wk_ctx* ctx, const double* u, double* out, int parts, void* stream);
/* M^{-1} K u (fused apply_inverse_mass(apply_K(u)))  operator.py:250-258 */
int wk_apply_minv_K(wk_ctx* ctx, const double* u, double* out, int parts, void* stream);
/* rhs(state) = -M^{-1} K u                      operator.py:268-272 */
int wk_rhs(wk_ctx* ctx, const double* u, double* out, void* stream);
/* apply_inverse_mass / apply_mass               operator.py:250-266 */
int wk_apply_inverse_mass(wk_ctx* ctx, const double* x, double* y, void* stream);
int wk_apply_mass(wk_ctx* ctx, const double* x, double* y, void* stream);
/* to_gauss_values / from_gauss_weighted         operator.py:276-284 */
int wk_to_gauss_values(wk_ctx* ctx, const double* x, double* y, void* stream);
int wk_from_gauss_weighted(wk_ctx* ctx, const double* x, double* y, void* stream);
/* apply_local_S(values, degree)                 operator.py:286-306 */
int wk_apply_local_S(wk_ctx* ctx, const double* x, double* y, int degree, void* stream);
/* resize_values(values, k_from, k_to)           operator.py:308-325 */
int wk_resize_values(wk_ctx* ctx, const double* x, double* y, int k_from, int k_to,
                     void* stream);

/* ---- fused steppers --------------------------------------------------- */
/* One low-storage RK stage (stepping.py:196-203) fused into the operator
 * epilogue: f = -M^{-1}K u_in; r = a r + dt f; u_out = u_in + b r.
 * a == 0 skips reading r.  u_out must not alias u_in. */
int wk_lsrk_stage(wk_ctx* ctx, const double* u_in, double* u_out, double* r, double a,
                  double b, double dt, void* stream);
/* The same stage with r_dead != 0 when the register is not read again before
 * it is overwritten: the LAST stage of a step (the next step's first stage
 * has a = 0, stepping.py:184-195 allocates r per step).  The streamed
 * kernels then skip the store of r (8 of the stage's 32 B/DoF); r is left
 * unspecified. */
int wk_lsrk_stage_ex(wk_ctx* ctx, const double* u_in, double* u_out, double* r, double a,
                     double b, double dt, int r_dead, void* stream);
/* Element-local Taylor sum (tck_evaluate, stepping.py:215-262); writes the
 * reference's mass-weighted GL result T. */
int wk_tck(wk_ctx* ctx, const double* w, double* t_out, double dt, int policy, int shift,
           void* stream);
/* One ADER step (ader_step, stepping.py:265-285) in two fused kernels.
 * U is updated in place; V and Y are caller scratch vectors (V unused for
 * WK_ADER). */
int wk_ader_step(wk_ctx* ctx, int variant, int policy, double* U, double* V, double* Y,
                 double dt, void* stream);
/* The two halves of wk_ader_step, for callers that exchange halos between
 * them (multi-GPU slabs): A reads U (+ U's neighbour faces for ADER-HDG) and
 * writes Y = M^{-1} T (and V = U - dt M^{-1}K U); B reads Y (+ its neighbour
 * faces) and V, and writes U = V - M^{-1} K Y (U - M^{-1} K Y for WK_ADER). */
int wk_ader_a(wk_ctx* ctx, int variant, int policy, const double* U, double* V, double* Y,
              double dt, void* stream);
int wk_ader_b(wk_ctx* ctx, int variant, double* U, const double* V, const double* Y,
              void* stream);

/* ---- fields around the time loop -------------------
 * Squared mass-weighted norm u . M u of a device state (state_norm,
 * stepping.py:321-324, is its square root); fused B sweeps + JxW-weighted
 * squares, deterministic fixed-order reduction; *out_sq is a DEVICE double. */
int wk_state_norm_sq(wk_ctx* ctx, const double* u, double* out_sq, void* stream);
/* Standing-mode state at the GL nodes of the multilinear vertex map
 * (initial_state, analytic.py:48-64): verts DEVICE (E, 2^d, d), vertex
 * v = sum_j a_j 2^j at corner (a_j); out DEVICE (E, d+1, (k+1)^d). */
int wk_mode_state(int d, int k, int64_t E, const double* verts, int m, double t, double c,
                  double rho, double* out, void* stream);
/* Squared L2 pressure error against the mode on the (k+1+n_extra)-point
 * Gauss rule (l2_pressure_error, analytic.py:67-93); *out_sq DEVICE. */
int wk_l2_pressure_error(int d, int k, int64_t E, const double* state, const double* verts,
                         int m, double t, double c, double rho, int n_extra, double* out_sq,
                         void* stream);

/* ---- curved geometry on the device ------------------
 * The GeometryCache arrays (precompute_geometry, mesh.py:307-334, with the
 * formulas of _volume_geometry / _face_geometry, mesh.py:245-286) from the
 * nodal coordinates of a degree-g map.  nodes: DEVICE (2, E, d, (g+1)^d),
 * direction 0 fastest: hi parts, then lo parts (double-double coordinates).
 * The point set is the tensor product of npts[m] points per direction;
 * val_hi/val_lo, der_hi/der_lo: HOST, per direction m the (npts[m], g+1) Lagrange value / derivative rows of the degree-g GL
 * basis, concatenated, as double-double pairs (row = hi + lo, evaluated in
 * extended precision on the host); wts: HOST (prod npts) point weights,
 * direction 0 fastest.  J, det, J^-1 and the normals are computed in
 * double-double and rounded once, so the result is reproducible to ~1 ulp
 * (the host builder does the same in long double).
 * face_axis < 0: volume -> inv_jac (E, d, d, P) = d xi_m / d x_i and
 *   jxw (E, P) = det J * w; stats (E, 3) (may be NULL) = per element
 *   max|J - J(point 0)|, max|offdiag J|, max|J| (cartesian_flag inputs).
 * face_axis = m >= 0, face_side = s: normal (E, d, P) outward unit normal,
 *   jxw (E, P) = |det J J^{-T} e_m| * w.
 * bad (DEVICE int, may be NULL) is set to 1 where det J <= 0. */
int wk_curved_metric(int d, int g, int64_t E, const double* nodes, const int32_t* npts,
                     const double* val_hi, const double* val_lo, const double* der_hi,
                     const double* der_lo, const double* wts, int face_axis,
                     int face_side, double* inv_jac, double* jxw, double* normal,
                     double* stats, int32_t* bad, void* stream);

/* Test hook: overwrite one device neighbour-table entry WITHOUT validation
 * (wk_ctx_create rejects out-of-range codes).  Used only to prove that the
 * checked build (libwk_b200_check.so, -DWK_CHECK) traps on a bad gather
 * index (tests/test_gpu_checked.py); never called by the product. */
int wk_debug_set_neighbor(wk_ctx* ctx, int64_t element, int face, int32_t value);

/* n_steps LSRK steps (lsrk_step, stepping.py:179-207, stage coefficients
 * a[0..n_stages), b[...], a[0] = 0) in ONE launch of one thread-block cluster
 * (<= 16 CTAs) whose shared memories hold the whole state; neighbour faces
 * through distributed shared memory, one cluster barrier per stage.  For
 * small Cartesian single-class affine meshes without halo (BASELINE config 1);
 * wk_lsrk_run_supported() says whether the context qualifies.  Bitwise equal
 * to n_steps x n_stages wk_lsrk_stage launches.  u_out may alias u_in. */
int wk_lsrk_run_supported(wk_ctx* ctx);
int wk_lsrk_run(wk_ctx* ctx, const double* u_in, double* u_out, int n_stages, const double* a,
                const double* b, double dt, int n_steps, void* stream);

/* Structured traversal of the persistent kernels (no reference counterpart:
 * a schedule, not arithmetic).  The element range [0, E) is viewed as
 * n_slow x n_blocks chunks of `chunk` consecutive elements (slow to fast);
 * full-mesh launches visit the chunks block-major (for each block, every
 * slow index), so the slow-axis neighbours of an element are streamed within
 * one chunk of it and their face values hit in L2.  For an x-fastest
 * structured mesh (nx, ny, nz): chunk = nx * by, n_blocks = ny / by,
 * n_slow = nz.  chunk = 0 restores mesh order.  Results are identical (the
 * per-element arithmetic does not depend on the order). */
int wk_set_tile_order(wk_ctx* ctx, int64_t chunk, int64_t n_slow, int64_t n_blocks);

/* ---- multi-GPU slab halo ------------------------------ */
/* Device pointer of the ghost buffer (G, d+1, n^(d-1)) the kernels read for
 * neighbour codes <= -2 (context-owned unless replaced). */
double* wk_ghost_buffer(wk_ctx* ctx);
/* Use a caller-owned device buffer (e.g. the NCCL receive tensor) instead. */
int wk_set_ghost_buffer(wk_ctx* ctx, double* ghost);
/* Pack face-node slices of `u` for export: entry i copies face (f_i) of local
 * element e_i into send[i] (shape (d+1, n^(d-1))).  export_elem / export_face
 * are host arrays of length n_export, copied once (set) and reused. */
int wk_set_halo_exports(wk_ctx* ctx, int64_t n_export, const int64_t* export_elem,
                        const int32_t* export_face);
int wk_pack_halo(wk_ctx* ctx, const double* u, double* send, void* stream);
/* Restrict the next fused/operator launches to local elements
 * [begin, begin+count) (interior/boundary overlap); count < 0 resets. */
int wk_set_element_range(wk_ctx* ctx, int64_t begin, int64_t count);
/* Tile-queue counter pair (0 or 1) used by the next launches: launches that
 * may run CONCURRENTLY on two streams (interior on the compute stream,
 * boundary on the halo stream) must use different slots. */
int wk_set_queue_slot(wk_ctx* ctx, int slot);

/* ---- host-side basis tables (no GPU needed) --------------------------- */
#define WK_TABLE_GAUSS_POINTS 0    /* (n)       quadrature.py:110-115 */
#define WK_TABLE_GAUSS_WEIGHTS 1
#define WK_TABLE_GL_POINTS 2       /* (n)       quadrature.py:118-154 */
#define WK_TABLE_GL_WEIGHTS 3
#define WK_TABLE_GL_TO_G 4         /* (n, n)    quadrature.py:239-254 */
#define WK_TABLE_G_TO_GL 5
#define WK_TABLE_D_GL 6            /* (n, n)    operator.py:111 */
#define WK_TABLE_D_CO 7            /* (n, n)    kernels.py:153-157 */
#define WK_TABLE_RESIZE 8          /* (k_to+1, k_from+1) operator.py:308-318 */
#define WK_TABLE_A_SPLIT 9         /* (n, n)    collapsed affine cell operator */
#define WK_TABLE_LIFT 10           /* (2, n)    M1^{-1} e_0, M1^{-1} e_{n-1} */
/* Writes the table for degree k (k_to used by WK_TABLE_RESIZE) into out;
 * returns the number of doubles written, or -1 on error. */
int wk_basis_table(int kind, int k, int k_to, double* out, int out_len);

#ifdef __cplusplus
}
#endif
#endif /* WAVEKERNEL_B200_H */
