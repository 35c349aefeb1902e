/*
 * pmgflow_b200.h -- C ABI of the B200-native (sm_100a, FP64) JFNK-pMG hot
 * path.  Plain pointers and sizes only; no torch / CUDA C++ types.
 *
 * The reference (pmgflow, pure Python/NumPy) has no FFI; its seams are
 * duck-typed Python callables.  Each entry point below
 * replaces one of those call sites; the ctypes binding a maintainer adds
 * is shown in INTEGRATION.md and lives in paper_2202_09733_b200/_lib.py.
 *
 * Conventions
 *  - Vectors are caller-owned DEVICE buffers (FP64, contiguous) in the
 *    reference layout: element e occupies [e*sz, (e+1)*sz), shaped
 *    (n, n, nvars) C-order, first index along eta (spatial.py:209-215).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Calls are asynchronous on that stream except the pmgb_status* and
 *    pmgb_sync calls.  One stream per discretization; not re-entrant.
 *  - Return value: 0 ok; > 0 a cudaError_t; < 0 a library error
 *    (see pmgb_error_string).
 *  - Non-physical states (rho <= 0 or p <= 0 at points, then traces,
 *    spatial.py:439-446, 506-510) do not abort the enqueued work; the
 *    first one seen is latched in a device status word and read back
 *    by pmgb_status (kind 1 = state, 2 = trace, with the smallest
 *    offending element of that residual evaluation).  Kind 3 = singular
 *    element-Jacobi block (newton_krylov.py:202-208); kind 4 = singular
 *    ILU0 pivot block (newton_krylov.py:340-343).
 */
#ifndef PMGFLOW_B200_H
#define PMGFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMGB_API __attribute__((visibility("default")))

typedef struct pmgb_disc pmgb_disc;

/* Discretization setup: replaces Discretization.__init__
 * (spatial.py:298-359) + element_geometry (mesh.py:322-395); uniform
 * degree 0..5.  All pointers are HOST arrays, copied to the device. */
typedef struct pmgb_disc_desc {
  int64_t n_elem;
  int32_t degree;             /* p; n = p + 1 points per direction       */
  int32_t kind;               /* 0 euler, 1 navier-stokes, 2 adv-diff    */
  double gamma, mu, kappa;    /* EquationSpec.gamma / .mu / .heat_cond.  */
  double adv_x, adv_y, diffusivity;
  const double* free_stream;  /* (nvars) EquationSpec.free_stream()      */
  const double* D;            /* (n, n) D[k][i] = l_i'(x_k)              */
  const double* eL;           /* (n) basis at xi = -1                    */
  const double* eR;           /* (n) basis at xi = +1                    */
  const double* lL;           /* (n) eL / w                              */
  const double* lR;           /* (n) eR / w                              */
  const double* xg;           /* (n) Gauss points                        */
  const double* geom;         /* (M, 20) see mesh.pack_geometry          */
  const int64_t* links;       /* (M, 4, 4) nb elem|-1, nb face, rev, is_left */
  const int32_t* tags;        /* (M, 4) boundary tag code, -1 interior    */
  int32_t riemann;            /* 0 Roe (reference), 1 Rusanov (option)   */
  int32_t viscous_scheme;     /* 0 BR1 (reference), 1 LDG (option)       */
  double wall_temperature;    /* T = p/rho on tag-3 "wall-isothermal"
                                 faces (option; EquationSpec.t_wall)      */
} pmgb_disc_desc;

PMGB_API int pmgb_disc_create(const pmgb_disc_desc* desc, pmgb_disc** out);
PMGB_API int pmgb_disc_destroy(pmgb_disc* d);
PMGB_API int64_t pmgb_disc_n_dofs(const pmgb_disc* d);
/* Residual kernel family of a context: 1 = the axis-aligned-rectangle
   path (fr_rect.cu; chosen at creation when every element qualifies),
   0 = the general bilinear path.  `want` < 0 only queries; 1 is honoured
   only when the mesh qualifies.  2 and 3 pin the rectangle path's
   four-kernel / two-kernel launch chain (1 takes the faster one per
   degree; for A/B runs and cross-checks).  Returns the path now in
   effect.  (No reference counterpart: every path implements
   spatial.py:501-570.)  On the rectangle path the state and operand
   arrays of pmgb_eval must be 32-byte aligned (error -6 otherwise). */
PMGB_API int pmgb_disc_residual_path(pmgb_disc* d, int32_t want);

/* R(q) -- replaces Discretization.residual (spatial.py:501-570). */
PMGB_API int pmgb_residual(pmgb_disc* d, const double* q, double* R, void* stream);

/* Fused residual evaluation with prologue q + eps*X (X may be NULL) and
 * an epilogue; replaces the vector algebra wrapped around residual()
 * at newton_krylov.py:71-76 (jfnk_matvec), :402-405 (PTC matvec),
 * time_integration.py:138-141 (stage_function), pmg.py:152-159
 * (LevelState.F / defect) and pmg.py:325-326 (pmg_solve outer F). */
enum {
  PMGB_EPI_R = 0,        /* out = R                                   */
  PMGB_EPI_F = 1,        /* out = s q - R                             */
  PMGB_EPI_DEFECT = 2,   /* out = (Sb - (s q - R)) + Se               */
  PMGB_EPI_JV = 3,       /* out = s X - (R(q + eps X) - R0) / eps     */
  PMGB_EPI_STAGE_F = 4,  /* out = (q - E) / adt - R                   */
  PMGB_EPI_STAGE_JV = 5, /* out = X/dtau + (F(q + eps X) - R0) / eps  */
  PMGB_EPI_NEG_R = 6,    /* out = -R                                  */
  PMGB_EPI_OUTER_F = 7,  /* out = (s q - R) - Se                      */
  PMGB_EPI_RK = 8        /* out = Q0 + alpha dtau_e[e] ((Sb - (s q - R)) + Se):
                          * one stage of the pseudo-transient RK smoother
                          * (not in the reference; BASELINE north star
                          * item 3); dtau_e from pmgb_rk_dtau          */
};
typedef struct pmgb_epilogue {
  int32_t mode;
  int32_t pad;
  double s, eps, adt, dtau, sb_scalar, se_scalar;
  const double* X;   /* device; JV modes           */
  const double* R0;  /* device; R0 (JV) / Fk (STAGE_JV) */
  const double* E;   /* device; explicit stage part */
  const double* Sb;  /* device or NULL -> sb_scalar */
  const double* Se;  /* device or NULL -> se_scalar */
  const double* Q0;      /* device; RK stage base state  */
  const double* dtau_e;  /* device (M); RK per-element pseudo-time step */
  double alpha;          /* RK stage coefficient */
} pmgb_epilogue;
PMGB_API int pmgb_eval(pmgb_disc* d, const double* q, const double* X, double eps,
                       const pmgb_epilogue* epi, double* out, void* stream);

/* Mixed-degree contexts (per-element degree map, p = 0..5; Euler / NS,
 * Roe or Rusanov, BR1): the reference's degree groups with mortar faces --
 * both traces interpolated (Pi) to the higher degree's face points, the
 * common values formed there and restricted (Gamma) back (spatial.py:
 * 468-497, 501-585).  `desc` as for pmgb_disc_create (its degree field is
 * ignored), `degrees` (M), `ops` (6, 66): per degree D (n x n packed)
 * then eL, eR, lL, lR, Gauss points at 36, 42, 48, 54, 60; `xfer`
 * (6 x 6 degree pairs [pH][pL], 2, 6 x 6): Pi (nH x nL) then Gamma
 * (nL x nH), row stride 6.  Vectors use the reference's flat layout
 * (element e at the offset of its degree's block size). */
typedef struct pmgb_mdisc pmgb_mdisc;
PMGB_API int pmgb_mdisc_create(const pmgb_disc_desc* desc, const int32_t* degrees, const double* ops,
                               const double* xfer, pmgb_mdisc** out);
PMGB_API int pmgb_mdisc_destroy(pmgb_mdisc* d);
PMGB_API int64_t pmgb_mdisc_n_dofs(const pmgb_mdisc* d);
/* R(q) with the fused epilogues of pmgb_eval (not PMGB_EPI_RK) */
PMGB_API int pmgb_mdisc_eval(pmgb_mdisc* d, const double* q, const double* X, double eps,
                             const pmgb_epilogue* epi, double* out, void* stream);
/* Frozen neighbour records (spatial.py:700-766) at own points, padded to
 * 6: rq (M,4,6,4) trace, rw (M,4,6,3) viscous variables, rf (M,4,6,4)
 * minus the neighbour's one-sided viscous flux; boundary faces untouched */
PMGB_API int pmgb_mdisc_freeze(pmgb_mdisc* d, const double* q, double* rq, double* rw, double* rf, void* stream);
/* element_residual (spatial.py:768-853) for B elements of degree p */
PMGB_API int pmgb_mdisc_element_residual(pmgb_mdisc* d, int32_t p, const int64_t* elems, int64_t B,
                                         const double* Q, const double* rq, const double* rw, const double* rf,
                                         double* out, void* stream);


/* Per-element spectral-radius estimate of dR/dq at state q for the RK
 * smoother's local pseudo-time step (PMGB_EPI_RK): lam (M doubles, device)
 *   = adv_coef max(|u|+c)/h_e + (p+1)^4 max(nu)/h_e^2,
 *   adv_coef = 2 sqrt(2) rho_p, rho_p the Bloch spectral radius of the 1-D
 *   upwind FR advection operator (operators.rk_adv_coef),
 *   h_e = 4 |det J(0,0)| / max(centre-line lengths).  No reference
 * counterpart (the reference's smoothers are EJ / MBNK, pmg.py:162-175). */
PMGB_API int pmgb_rk_lambda(pmgb_disc* d, const double* q, double adv_coef, double* lam, void* stream);

/* RK local pseudo-time steps dtau[e] = cfl / (s + lam[e]) (M elements,
 * device buffers), once per smoothing sweep set. */
PMGB_API int pmgb_rk_dtau(int64_t M, const double* lam, double s, double cfl, double* dtau, void* stream);

/* (shift I - dR/dq) X ~ shift X - (R(q+eps X) - R0)/eps
 * -- newton_krylov.py:71-76. */
PMGB_API int pmgb_jfnk_matvec(pmgb_disc* d, const double* X, const double* q, const double* R0,
                              double shift, double eps, double* out, void* stream);

/* freeze (spatial.py:700-766): face traces qtr (M,4,n,nv) and one-sided
 * viscous normal fluxes fvn (M,4,n,nv) of state q; every frozen record of
 * the reference is a gather from these two arrays. fvn unused (may be
 * NULL) for inviscid kinds. */
PMGB_API int pmgb_freeze(pmgb_disc* d, const double* q, double* qtr, double* fvn, void* stream);

/* element_residual (spatial.py:768-853) for B instances (elems[b], Q[b]),
 * neighbours frozen at (qtr, fvn).  elems: device int64 (B). */
PMGB_API int pmgb_element_residual(pmgb_disc* d, const int64_t* elems, int64_t B, const double* Q,
                                   const double* qtr, const double* fvn, double* out, void* stream);

/* assemble_element_blocks (newton_krylov.py:157-210): FD blocks of
 * shift I - dR_e/dq_e (eps perturbations of the frozen element-local
 * residual) stored column-major per element in blocksT (M, sz, sz).  If
 * XT is not NULL the blocks are also inverted (np.linalg.inv at
 * newton_krylov.py:201) by Gauss-Jordan with implicit partial pivoting:
 * XT (M, sz, sz) receives the in-place factor column-major and perm
 * (M, 2*sz) uint8 the pivot rows p and their inverse q, such that
 * B^-1[i][j] = X[p_i][q_j].  XT may equal blocksT.  A singular block
 * latches status kind 3 (RuntimeError at newton_krylov.py:202-208). */
PMGB_API int pmgb_blocks_assemble(pmgb_disc* d, const double* q, double shift, double eps,
                                  double* blocksT, double* XT, uint8_t* perm, void* stream);
PMGB_API int pmgb_blocks_invert(int64_t n_elem, int32_t sz, const double* blocksT, double* XT, uint8_t* perm,
                                void* stream);

/* assemble_sparse_blocks (newton_krylov.py:281-311) with coupling_block
 * (:254-278) and Discretization.neighbor_face_record / element_residual
 * face_override (spatial.py:768-903): the block-CSR values of
 * A = shift I - dR/dq on the element-adjacency pattern, every block
 * column-major (blocks[k][c][r] = A_k[r][c]).  The host supplies the
 * pattern: diag_slot[e] = CSR slot of (e, e); pairs (pair_e, pair_f) are
 * the interior (element, face) couplings in the reference's accumulation
 * order, grouped into nwaves waves (pairs [wave_ptr[w], wave_ptr[w+1]))
 * in which every target slot pair_slot appears at most once; pair_add = 1
 * adds onto the slot (second face of a periodic pair, or a self-coupling
 * onto the diagonal).  wave_ptr is a HOST array of nwaves+1 offsets; all
 * other arrays are device arrays; q is the level state. */
PMGB_API int pmgb_sparse_assemble(pmgb_disc* d, const double* q, double shift, double eps, double* blocks,
                                  const int32_t* diag_slot, int64_t npairs, const int32_t* pair_e,
                                  const int8_t* pair_f, const int32_t* pair_slot, const int8_t* pair_add,
                                  const int64_t* wave_ptr, int32_t nwaves, void* stream);

/* SparseBlockMatrix.matvec (newton_krylov.py:243-251): y_i = sum over the
 * row's CSR entries k of A_k x_{indices[k]}, blocks column-major, int32
 * device CSR arrays. */
PMGB_API int pmgb_sparse_matvec(int64_t n_rows, int32_t sz, const int32_t* indptr, const int32_t* indices,
                                const double* blocks, const double* x, double* y, void* stream);

/* ilu0_factor (newton_krylov.py:319-345): block ILU with zero fill, in
 * place on F (a copy of the CSR values), level-scheduled: level L holds the
 * rows level_rows[level_ptr[L] .. level_ptr[L+1]) of the lower-neighbour
 * DAG (level_diag = their diagonal CSR slots); every row performs the
 * reference's block operations in its order.  The pivot-block inverses
 * are stored as Gauss-Jordan factors (DX, DP) like the EJ blocks; a
 * singular pivot block latches status kind 4 (RuntimeError "singular ILU0
 * pivot block at element i").  level_ptr is a HOST array. */
PMGB_API int pmgb_ilu0_factor(int64_t n_rows, int32_t sz, const int32_t* indptr, const int32_t* indices,
                               double* F, double* DX, uint8_t* DP, int32_t n_levels, const int64_t* level_ptr,
                               const int32_t* level_rows, const int32_t* level_diag, void* stream);

/* ilu0_apply (newton_krylov.py:348-368): forward sweep with the unit lower
 * factor over the lower-DAG levels (into y), backward sweep with the upper
 * factor and the pivot inverses over the upper-DAG levels (into out).
 * lo_ptr / up_ptr are HOST arrays. */
PMGB_API int pmgb_ilu0_apply(int64_t n_rows, int32_t sz, const int32_t* indptr, const int32_t* indices,
                              const double* F, const double* DX, const uint8_t* DP, int32_t n_lo,
                              const int64_t* lo_ptr, const int32_t* lo_rows, int32_t n_up, const int64_t* up_ptr,
                              const int32_t* up_rows, const double* x, double* y, double* out, void* stream);

/* compute_forces (spatial.py:633-695): per wall (element, face) pair the
 * integrated force 2-vector  sum_k w_k face_jac (p n - tau n)  at state q
 * (traces and BR1 gradients recomputed on the device), out (n_wall, 2);
 * the caller sums the pairs (Fd, Fl) and forms the coefficients.  weights
 * = the n Gauss weights (host array).  Flow kinds only (-5 otherwise). */
PMGB_API int pmgb_wall_forces(pmgb_disc* d, const double* q, int64_t n_wall, const int32_t* wall_e,
                              const int8_t* wall_f, const double* weights, double* out, void* stream);

/* The same ilu0_apply as ONE cooperative launch: a co-resident grid walks
 * the forward then the backward levels with a global barrier between
 * levels (same per-row arithmetic).  row_entries (n_rows, 8, 2) int32:
 * the (CSR slot, column) of each row's lower (first 4) and upper (last 4)
 * blocks in column order, -1 padded.  Level pointers are DEVICE int32
 * arrays here; barrier = 2 device uint32 words of scratch; max_level_rows
 * = the largest level (caps the grid). */
PMGB_API int pmgb_ilu0_apply_fused(int32_t sz, const int32_t* row_entries, const double* F,
                                    const double* DX, const uint8_t* DP, int32_t n_lo, const int32_t* lo_ptr_dev,
                                    const int32_t* lo_rows, int32_t n_up, const int32_t* up_ptr_dev,
                                    const int32_t* up_rows, int32_t max_level_rows, const double* x, double* y,
                                    double* out, uint32_t* barrier, void* stream);

/* BlockJacobian.apply / ej_apply (newton_krylov.py:166-171, 213-214):
 * y_e = B_e^-1 x_e from (XT, perm).  pmgb_ej_update: out = base + omega *
 * B^-1 d (smooth_ej, pmg.py:162-164); out may alias base. */
PMGB_API int pmgb_ej_apply(int64_t n_elem, int32_t sz, const double* XT, const uint8_t* perm, const double* x,
                           double* y, void* stream);
PMGB_API int pmgb_ej_update(int64_t n_elem, int32_t sz, const double* XT, const uint8_t* perm, const double* d,
                            double omega, const double* base, double* out, void* stream);

/* Option pmg.block_precision = fp32 (not in the reference, whose blocks are
 * float64): the factor XT stored in FP32 (round to nearest), applied with
 * FP64 arithmetic -- half the bytes of the step's dominant HBM stream and
 * of the per-level block memory.  Same (perm, layout) as the FP64 calls. */
PMGB_API int pmgb_blocks_demote(int64_t n_elem, int32_t sz, const double* XT, float* XT32, void* stream);
PMGB_API int pmgb_ej_apply_f32(int64_t n_elem, int32_t sz, const float* XT32, const uint8_t* perm,
                               const double* x, double* y, void* stream);
PMGB_API int pmgb_ej_update_f32(int64_t n_elem, int32_t sz, const float* XT32, const uint8_t* perm,
                                const double* d, double omega, const double* base, double* out, void* stream);

/* pMG transfers (pmg.py:117-136).  T is a HOST (n_out x n_in) matrix:
 * Gamma for restriction, Pi for prolongation.
 *   pmgb_transfer:     dst = (T (x) T) (src - src_base)   [src_base may be NULL]
 *   accumulate != 0:   dst += ...                          (prolong + add) */
PMGB_API int pmgb_transfer(int64_t n_elem, int32_t nvars, int32_t n_in, int32_t n_out, const double* T,
                           const double* src, const double* src_base, double* dst, int32_t accumulate,
                           void* stream);

/* Deterministic reductions and Arnoldi (newton_krylov.py:79-151). */
PMGB_API int pmgb_dot(int64_t n, const double* x, const double* y, double* result_dev, void* stream);
PMGB_API int pmgb_nrm2(int64_t n, const double* x, double* result_dev, void* stream);
/* MGS of w against rows 0..j of V (row stride ld): H_dev[0..j+1] gets
 * column j of the Hessenberg matrix, V[j+1] = w / H[j+1] when
 * H[j+1] > thresh, *finite_dev = 1 if w entered with a non-finite. */
PMGB_API int pmgb_mgs(int64_t n, double* V, int64_t ld, int32_t j, double* w, double* H_dev, double thresh,
                      int32_t* finite_dev, void* stream);
/* The partitioned Arnoldi step as separate passes over a
 * rank's owned range, so each partial dot can be all-reduced in-stream
 * between them: pmgb_mgs_pass does w -= (*hprev) Vprev (Vprev may be NULL)
 * then *out = Vnext . w (first != 0: reset the finite flag and check w as
 * it enters; finite_dev may be NULL); pmgb_normalize_sqrt sets
 * *h = sqrt(*h) (the all-reduced w . w) and V_{j+1} = w / *h if > thresh. */
PMGB_API int pmgb_mgs_pass(int64_t n, double* w, const double* Vprev, const double* hprev, const double* Vnext,
                           double* out, int32_t first, int32_t* finite_dev, void* stream);
PMGB_API int pmgb_normalize_sqrt(int64_t n, const double* w, double* h_dev, double thresh, double* v,
                                 void* stream);
/* Classical Gram-Schmidt with reorthogonalisation (option gmres.ortho =
 * cgs2; the reference orthogonalises by MGS, newton_krylov.py:119-123):
 * pmgb_multidot sets out_dev[c] = V_c . w for c < k <= 256 (rows of V at
 * stride ld; deterministic order; *finite_dev |= non-finite w, may be
 * NULL) and pmgb_gemv_sub does w -= V[0:k]^T y_dev. */
PMGB_API int pmgb_multidot(int64_t n, const double* V, int64_t ld, int32_t k, const double* w, double* out_dev,
                           int32_t* finite_dev, void* stream);
PMGB_API int pmgb_gemv_sub(int64_t n, int32_t k, const double* V, int64_t ld, const double* y_dev, double* w,
                           void* stream);
/* out = sum_i c[i] x[i], k <= 8, c and the pointer array on the HOST. */
PMGB_API int pmgb_lincomb(int64_t n, int32_t k, const double* c, const double* const* xs, double* out,
                          void* stream);
/* out = V[0:k]^T y, y on the device (k <= 28992). */
PMGB_API int pmgb_gemv_t(int64_t n, int32_t k, const double* V, int64_t ld, const double* y_dev, double* out,
                         void* stream);
/* *flag_dev = any(x != 0) */
PMGB_API int pmgb_any_nonzero(int64_t n, const double* x, int32_t* flag_dev, void* stream);

/* Status word (non-physical / singular), synchronising. */
PMGB_API int pmgb_status(void* stream, int32_t* kind, int64_t* element, int32_t clear);
PMGB_API int pmgb_status_clear(void* stream);
PMGB_API int pmgb_sync(void* stream);
PMGB_API const char* pmgb_error_string(int code);
/* FP64 throughput probe: `blocks` CTAs x 256 threads x 8 DFMA chains x
 * iters (2 flops each); the FP64 roof for bench.py's roofline. */
PMGB_API int pmgb_probe_fp64(int64_t iters, int32_t blocks, double* out_dev, void* stream);
/* Build/version tag and a count of kernel launches issued (diagnostics). */
PMGB_API const char* pmgb_version(void);
PMGB_API int64_t pmgb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PMGFLOW_B200_H */
