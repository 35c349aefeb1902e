// extern "C" boundary of libpmgflow_b200.so -- see include/pmgflow_b200.h.
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/pmgflow_b200.h"
#include "pmgb_internal.cuh"

namespace pmgb {
int launch_inverse(int64_t M, int SZ, const double* BT, double* XT, uint8_t* perm, cudaStream_t st, Status* stp,
                   const int* in_slot = nullptr, const int* out_idx = nullptr, int bad_kind = 3);
int launch_ilu_level(int64_t n, int SZ, const int* rows, const int* indptr, const int* indices, double* F,
                     const double* DX, const uint8_t* DP, cudaStream_t st);
int launch_ilu_sweep(int backward, int64_t n, int SZ, const int* rows, const int* indptr, const int* indices,
                     const double* F, const double* DX, const uint8_t* DP, const double* in, double* out,
                     cudaStream_t st);
int launch_ilu_persistent(int SZ, int n_lo, const int* lo_ptr, const int* lo_rows, int n_up, const int* up_ptr,
                          const int* up_rows, const int* ent, const double* F,
                          const double* DX, const uint8_t* DP, const double* x, double* y, double* out,
                          unsigned* bar, int max_rows, cudaStream_t st);
int launch_block_gemv(int64_t M, int SZ, const double* XT, const uint8_t* perm, const double* x, double omega,
                      const double* base, double* out, cudaStream_t st);
int launch_block_gemv_f32(int64_t M, int SZ, const float* XT, const uint8_t* perm, const double* x, double omega,
                          const double* base, double* out, cudaStream_t st);
int launch_demote(int64_t n, const double* src, float* dst, cudaStream_t st);
int launch_transfer(int64_t M, int nv, int nin, int nout, const double* T, const double* src,
                    const double* src_base, double* dst, int accumulate, cudaStream_t st);
int launch_dot(int64_t n, const double* x, const double* y, double* out, int do_sqrt, cudaStream_t st);
int launch_mgs(int64_t n, double* V, int64_t ld, int j, double* w, double* H, double thresh, int* finite_flag,
               cudaStream_t st);
int launch_mgs_pass(int64_t n, double* w, const double* Vprev, const double* hprev, const double* Vnext,
                    double* out, int first, int* finite_flag, cudaStream_t st);
int launch_normalize_sqrt(int64_t n, const double* w, double* h, double thresh, double* v, cudaStream_t st);
int launch_lincomb(int64_t n, int k, const double* c, const double* const* xs, double* out, cudaStream_t st);
int launch_rk_dtau(int64_t M, const double* lam, double s, double cfl, double* dtau, cudaStream_t st);
int launch_gemv_t(int64_t n, int k, const double* V, int64_t ld, const double* y, double* out, cudaStream_t st);
int launch_any_nonzero(int64_t n, const double* x, int* flag_dev, cudaStream_t st);
int launch_multidot(int64_t n, const double* V, int64_t ld, int k, const double* w, double* out, int* flag,
                    cudaStream_t st);
int launch_gemv_sub(int64_t n, int k, const double* V, int64_t ld, const double* y, double* w, cudaStream_t st);
int launch_probe_fp64(int64_t iters, int blocks, double* out, cudaStream_t st);
Status* status_ptr();
int* bad_ptr();

// mixed-degree path (fr_mixed.cu)
struct MixDev {
  int64_t M;
  int kind;
  const int8_t* deg;
  const int64_t* off;
  const int64_t* poff;
  const double* geom;
  const int2* link;
  const double* ops;
  const double* xfer;
  int64_t nface;
  const int4* faces;
};
struct MixGroups {
  const int* elems[6];
  int64_t cnt[6];
};
int mx_residual(const FrConst& C, const MixDev& m, const MixGroups& gr, const double* q, const double* X,
                double eps, const Epi& ep, double* qtr, double* fci, double* wh, double* grad, double* fvn,
                double* fcv, double* out, int* bad, Status* stp, cudaStream_t st);
int mx_records(const FrConst& C, const MixDev& m, const double* qtr, const double* fvn, double* rq, double* rw,
               double* rf, cudaStream_t st);
int mx_local(const FrConst& C, const MixDev& m, int p, const int64_t* elems, int64_t B, const double* Q,
             const double* rq, const double* rw, const double* rf, double* out, cudaStream_t st);
}  // namespace pmgb

using namespace pmgb;

struct pmgb_disc {
  DiscDev d;
};

static std::atomic<int64_t> g_launches{0};
static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

extern "C" {

PMGB_API const char* pmgb_version(void) { return "pmgflow_b200 0.1 sm_100a fp64"; }
PMGB_API int64_t pmgb_launch_count(void) { return g_launches.load(); }

PMGB_API const char* pmgb_error_string(int code) {
  if (code == 0) return "ok";
  if (code > 0) return cudaGetErrorString((cudaError_t)code);
  switch (code) {
    case -1: return "invalid argument";
    case -2: return "unsupported polynomial degree (0..5)";
    case -3: return "unsupported equation kind";
    case -4: return "mesh too large for one device context (face offsets exceed 2^31)";
    case -5: return "forces are only defined for flow equations";
    case -6: return "state / operand arrays must be 32-byte aligned (256-bit accesses)";
    case -1000: return "no kernel instance for this degree/kind";
    case -1001: return "vector count out of range";
  }
  return "unknown pmgflow_b200 error";
}

// Rectangle fast path (fr_rect.cu): taken when every element is an
// axis-aligned rectangle whose geometry record has exactly zero cross
// metric terms, axis-aligned unit normals and face_jac equal to the
// half-widths -- then the reference's metric expressions reduce to
// per-element constants with no rounding of their own.  Builds the
// unique-face list (sorted by owner element) and the face records.
static int setup_rect(const pmgb_disc_desc* desc, DiscDev& d) {
  d.has_rect = 0;
  if (!rect_supported(d.p, d.kind) || d.M == 0) return 0;
  const char* env = std::getenv("PMGB_RECT");  // PMGB_RECT=0: general kernels only (A/B)
  if (env != nullptr && env[0] == '0') return 0;
  const double* G = desc->geom;
  std::vector<double2> rg((size_t)d.M);
  for (int64_t e = 0; e < d.M; ++e) {
    const double* g = G + e * 20;
    const double a0 = g[0], d0 = g[6];
    const bool ok = g[1] == 0.0 && g[2] == 0.0 && g[3] == 0.0 && g[4] == 0.0 && g[5] == 0.0 && g[7] == 0.0 &&
                    a0 > 0.0 && d0 > 0.0 && g[8] == 0.0 && g[9] == -1.0 && g[10] == 1.0 && g[11] == 0.0 &&
                    g[12] == 0.0 && g[13] == 1.0 && g[14] == -1.0 && g[15] == 0.0 && g[16] == a0 &&
                    g[18] == a0 && g[17] == d0 && g[19] == d0;
    if (!ok) return 0;
    rg[(size_t)e] = make_double2(1.0 / a0, 1.0 / d0);
  }
  std::vector<int4> faces;
  faces.reserve((size_t)d.M * 2 + 16);
  std::vector<int> fslot((size_t)d.M * 4, -1);
  for (int64_t e = 0; e < d.M; ++e)
    for (int f = 0; f < 4; ++f) {
      const int64_t* r = desc->links + (e * 4 + f) * 4;
      const bool bnd = r[0] < 0;
      if (!bnd && !(r[3] & 1)) continue;  // the L side owns the face
      const int tag = desc->tags[e * 4 + f];
      int4 v;
      v.x = (int)e;
      v.y = f | ((int)(r[2] & 1) << 2) | ((int)bnd << 3) | ((tag < 0 ? 0 : tag & 15) << 4);
      v.z = bnd ? -1 : (int)r[0];
      v.w = bnd ? 0 : (int)r[1];
      const int phi = (int)faces.size();
      faces.push_back(v);
      fslot[(size_t)e * 4 + f] = phi;
      if (!bnd) fslot[(size_t)r[0] * 4 + r[1]] = phi;
    }
  for (int v : fslot)
    if (v < 0) return -1;
  RectDev& R = d.rect;
  R.nface = (int64_t)faces.size();
  const int n = d.p + 1;
  cudaError_t err = cudaMalloc(&R.faces, sizeof(int4) * faces.size());
  if (!err) err = cudaMalloc(&R.fslot, sizeof(int) * fslot.size());
  if (!err) err = cudaMalloc(&R.rgeo, sizeof(double2) * rg.size());
  if (!err) err = cudaMalloc(&R.frec, sizeof(double) * 12 * (size_t)R.nface * n);
  if (!err) err = cudaMalloc(&R.wh, sizeof(double) * 3 * 4 * (size_t)d.M * n);
  if (!err) err = cudaMalloc(&R.fc, sizeof(double) * 4 * 4 * (size_t)d.M * n);
  if (!err) err = cudaMemcpy(R.faces, faces.data(), sizeof(int4) * faces.size(), cudaMemcpyHostToDevice);
  if (!err) err = cudaMemcpy(R.fslot, fslot.data(), sizeof(int) * fslot.size(), cudaMemcpyHostToDevice);
  if (!err) err = cudaMemcpy(R.rgeo, rg.data(), sizeof(double2) * rg.size(), cudaMemcpyHostToDevice);
  if (err) return (int)err;
  d.has_rect = 1;
  return 0;
}

PMGB_API int pmgb_disc_create(const pmgb_disc_desc* desc, pmgb_disc** out) {
  if (!desc || !out) return -1;
  if (desc->degree < 0 || desc->degree > 5) return -2;
  if (desc->kind < 0 || desc->kind > 2) return -3;
  if (desc->riemann < 0 || desc->riemann > 1 || desc->viscous_scheme < 0 || desc->viscous_scheme > 1) return -1;
  if (desc->n_elem * 4 * (desc->degree + 1) * 4 >= ((int64_t)1 << 31)) return -4;  // 32-bit face offsets
  pmgb_disc* h = new pmgb_disc();
  DiscDev& d = h->d;
  std::memset(&d.C, 0, sizeof(d.C));
  d.p = desc->degree;
  const int n = d.p + 1;
  d.kind = desc->kind == 0 ? K_EULER : desc->kind == 1 ? K_NS : (desc->diffusivity > 0.0 ? K_ADVD : K_ADV);
  d.nv = desc->kind == 2 ? 1 : 4;
  d.M = desc->n_elem;
  d.n_dofs = d.M * n * n * d.nv;
  for (int i = 0; i < n * n; ++i) d.C.D[i] = desc->D[i];
  for (int i = 0; i < n; ++i) {
    d.C.eL[i] = desc->eL[i];
    d.C.eR[i] = desc->eR[i];
    d.C.lL[i] = desc->lL[i];
    d.C.lR[i] = desc->lR[i];
    d.C.xg[i] = desc->xg[i];
  }
  for (int v = 0; v < d.nv; ++v) d.C.qinf[v] = desc->free_stream[v];
  d.C.gamma = desc->gamma;
  d.C.mu = desc->mu;
  d.C.kappa = desc->kappa;
  d.C.adv_x = desc->adv_x;
  d.C.adv_y = desc->adv_y;
  d.C.diff = desc->diffusivity;
  d.C.riemann = desc->riemann;
  d.C.ldg = desc->viscous_scheme;
  d.C.twall = desc->wall_temperature;
  std::vector<int2> lk((size_t)d.M * 4);
  for (int64_t e = 0; e < d.M; ++e) {
    for (int f = 0; f < 4; ++f) {
      const int64_t* r = desc->links + (e * 4 + f) * 4;
      const int tag = desc->tags[e * 4 + f];
      int2 v;
      v.x = (int)r[0];
      const int face = r[0] >= 0 ? (int)r[1] : 0;
      v.y = (face & 3) | ((int)(r[2] & 1) << 2) | ((int)(r[3] & 1) << 3) | ((tag < 0 ? 0 : tag & 15) << 4);
      lk[(size_t)e * 4 + f] = v;
    }
  }
  const size_t face_bytes = sizeof(double) * (size_t)d.M * 4 * n * d.nv;
  cudaError_t err = cudaSuccess;
  err = cudaMalloc(&d.geom, sizeof(double) * 20 * (size_t)d.M);
  if (!err) err = cudaMalloc(&d.link, sizeof(int2) * 4 * (size_t)d.M);
  if (!err) err = cudaMalloc(&d.qtr, face_bytes);
  if (!err) err = cudaMalloc(&d.fvn, face_bytes);
  if (!err) err = cudaMalloc(&d.qp, sizeof(double) * (size_t)d.n_dofs);
  // gradients: per CTA block, k_fvn's padded planes (fr_grad_scratch_doubles)
  if (!err) err = cudaMalloc(&d.grad, sizeof(double) * fr_grad_scratch_doubles(d.p, d.kind, d.M));
  if (!err) err = cudaMemcpy(d.geom, desc->geom, sizeof(double) * 20 * (size_t)d.M, cudaMemcpyHostToDevice);
  if (!err) err = cudaMemcpy(d.link, lk.data(), sizeof(int2) * 4 * (size_t)d.M, cudaMemcpyHostToDevice);
  if (err) {
    pmgb_disc_destroy(h);
    return (int)err;
  }
  d.mesh.M = d.M;
  d.mesh.geom = d.geom;
  d.mesh.link = d.link;
  err = (cudaError_t)setup_rect(desc, d);
  if (err) {
    pmgb_disc_destroy(h);
    return (int)err;
  }
  *out = h;
  return 0;
}

PMGB_API int pmgb_disc_destroy(pmgb_disc* h) {
  if (!h) return 0;
  cudaFree(h->d.geom);
  cudaFree(h->d.link);
  cudaFree(h->d.qtr);
  cudaFree(h->d.fvn);
  cudaFree(h->d.qp);
  cudaFree(h->d.grad);
  cudaFree(h->d.rect.faces);
  cudaFree(h->d.rect.fslot);
  cudaFree(h->d.rect.rgeo);
  cudaFree(h->d.rect.frec);
  cudaFree(h->d.rect.wh);
  cudaFree(h->d.rect.fc);
  delete h;
  return 0;
}

PMGB_API int64_t pmgb_disc_n_dofs(const pmgb_disc* h) { return h ? h->d.n_dofs : -1; }

// ---------------------------------------------------------------------------
// mixed-degree contexts (fr_mixed.cu)

struct pmgb_mdisc {
  FrConst C;
  MixDev m;
  MixGroups gr;
  int8_t* deg = nullptr;
  int64_t *off = nullptr, *poff = nullptr;
  double *geom = nullptr, *ops = nullptr, *xfer = nullptr;
  int2* link = nullptr;
  int4* faces = nullptr;
  int* elems = nullptr;
  double *qtr = nullptr, *fci = nullptr, *wh = nullptr, *grad = nullptr, *fvn = nullptr, *fcv = nullptr;
  int64_t n_dofs = 0;
};

PMGB_API int pmgb_mdisc_destroy(pmgb_mdisc* h) {
  if (!h) return 0;
  for (void* p : {(void*)h->deg, (void*)h->off, (void*)h->poff, (void*)h->geom, (void*)h->ops, (void*)h->xfer,
                  (void*)h->link, (void*)h->faces, (void*)h->elems, (void*)h->qtr, (void*)h->fci, (void*)h->wh,
                  (void*)h->grad, (void*)h->fvn, (void*)h->fcv})
    cudaFree(p);
  delete h;
  return 0;
}

PMGB_API int pmgb_mdisc_create(const pmgb_disc_desc* desc, const int32_t* degrees, const double* ops,
                               const double* xfer, pmgb_mdisc** out) {
  if (!desc || !degrees || !ops || !xfer || !out) return -1;
  if (desc->kind != 0 && desc->kind != 1) return -3;  // Euler / Navier-Stokes
  if (desc->viscous_scheme != 0) return -1;            // BR1 (the reference's scheme)
  const int64_t M = desc->n_elem;
  pmgb_mdisc* h = new pmgb_mdisc();
  std::memset(&h->C, 0, sizeof(h->C));
  FrConst& C = h->C;
  for (int v = 0; v < 4; ++v) C.qinf[v] = desc->free_stream[v];
  C.gamma = desc->gamma;
  C.mu = desc->mu;
  C.kappa = desc->kappa;
  C.riemann = desc->riemann;
  C.twall = desc->wall_temperature;
  std::vector<int8_t> deg((size_t)M);
  std::vector<int64_t> off((size_t)M + 1, 0), poff((size_t)M + 1, 0);
  std::vector<std::vector<int>> groups(6);
  for (int64_t e = 0; e < M; ++e) {
    const int p = degrees[e];
    if (p < 0 || p > 5) {
      delete h;
      return -2;
    }
    deg[(size_t)e] = (int8_t)p;
    off[(size_t)e + 1] = off[(size_t)e] + 4 * (p + 1) * (p + 1);
    poff[(size_t)e + 1] = poff[(size_t)e] + (p + 1) * (p + 1);
    groups[p].push_back((int)e);
  }
  h->n_dofs = off[(size_t)M];
  std::vector<int2> lk((size_t)M * 4);
  std::vector<int4> faces;
  for (int64_t e = 0; e < M; ++e)
    for (int f = 0; f < 4; ++f) {
      const int64_t* r = desc->links + (e * 4 + f) * 4;
      const int tag = desc->tags[e * 4 + f];
      const bool bnd = r[0] < 0;
      int2 v;
      v.x = (int)r[0];
      v.y = (bnd ? 0 : (int)(r[1] & 3)) | ((int)(r[2] & 1) << 2) | ((int)(r[3] & 1) << 3) |
            ((tag < 0 ? 0 : tag & 15) << 4);
      lk[(size_t)e * 4 + f] = v;
      if (!bnd && !(r[3] & 1)) continue;
      int4 fa;
      fa.x = (int)e;
      fa.y = f | ((int)(r[2] & 1) << 2) | ((int)bnd << 3) | ((tag < 0 ? 0 : tag & 15) << 4);
      fa.z = bnd ? -1 : (int)r[0];
      fa.w = bnd ? 0 : (int)r[1];
      faces.push_back(fa);
    }
  std::vector<int> elems;
  int64_t gstart[6];
  for (int p = 0; p < 6; ++p) {
    gstart[p] = (int64_t)elems.size();
    elems.insert(elems.end(), groups[p].begin(), groups[p].end());
    h->gr.cnt[p] = (int64_t)groups[p].size();
  }
  const size_t fpad = sizeof(double) * (size_t)M * 4 * 6;
  cudaError_t err = cudaSuccess;
  auto up = [&](auto** dst, const void* src, size_t bytes) {
    if (err) return;
    err = cudaMalloc((void**)dst, bytes > 0 ? bytes : 16);
    if (!err && bytes) err = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  up(&h->deg, deg.data(), deg.size());
  up(&h->off, off.data(), sizeof(int64_t) * off.size());
  up(&h->poff, poff.data(), sizeof(int64_t) * poff.size());
  up(&h->geom, desc->geom, sizeof(double) * 20 * (size_t)M);
  up(&h->ops, ops, sizeof(double) * 6 * 66);
  up(&h->xfer, xfer, sizeof(double) * 36 * 2 * 36);
  up(&h->link, lk.data(), sizeof(int2) * lk.size());
  up(&h->faces, faces.data(), sizeof(int4) * faces.size());
  up(&h->elems, elems.data(), sizeof(int) * elems.size());
  if (!err) err = cudaMalloc(&h->qtr, fpad * 4);
  if (!err) err = cudaMalloc(&h->fci, fpad * 4);
  if (!err) err = cudaMalloc(&h->fvn, fpad * 4);
  if (!err) err = cudaMalloc(&h->fcv, fpad * 4);
  if (!err) err = cudaMalloc(&h->wh, fpad * 3);
  if (!err) err = cudaMalloc(&h->grad, sizeof(double) * 6 * (size_t)(poff[(size_t)M] + 1));
  if (err) {
    pmgb_mdisc_destroy(h);
    return (int)err;
  }
  for (int p = 0; p < 6; ++p) h->gr.elems[p] = h->elems + gstart[p];
  h->m = MixDev{M, desc->kind == 0 ? K_EULER : K_NS, h->deg, h->off, h->poff, h->geom, h->link, h->ops, h->xfer,
                (int64_t)faces.size(), h->faces};
  *out = h;
  return 0;
}

PMGB_API int64_t pmgb_mdisc_n_dofs(const pmgb_mdisc* h) { return h ? h->n_dofs : -1; }

PMGB_API int pmgb_mdisc_eval(pmgb_mdisc* h, const double* q, const double* X, double eps, const pmgb_epilogue* e,
                             double* out, void* stream) {
  if (!h || !q || !out || !e) return -1;
  if (e->mode == PMGB_EPI_RK) return -1;
  Epi ep;
  ep.mode = e->mode;
  ep.s = e->s;
  ep.eps = e->eps;
  ep.adt = e->adt;
  ep.dtau = e->dtau;
  ep.sb_scalar = e->sb_scalar;
  ep.se_scalar = e->se_scalar;
  ep.X = e->X;
  ep.R0 = e->R0;
  ep.E = e->E;
  ep.Sb = e->Sb;
  ep.Se = e->Se;
  ep.Q0 = nullptr;
  ep.dtau_e = nullptr;
  ep.alpha = 0.0;
  ep.npe = 0;
  int groups = 0;
  for (int p = 0; p < 6; ++p) groups += h->gr.cnt[p] ? 1 : 0;
  g_launches += groups * (h->m.kind == K_NS ? 3 : 2) + (h->m.kind == K_NS ? 2 : 1) + 1;
  return mx_residual(h->C, h->m, h->gr, q, X, eps, ep, h->qtr, h->fci, h->wh, h->grad, h->fvn, h->fcv, out,
                     bad_ptr(), status_ptr(), S(stream));
}

PMGB_API int pmgb_mdisc_freeze(pmgb_mdisc* h, const double* q, double* rq, double* rw, double* rf, void* stream) {
  if (!h || !q || !rq) return -1;
  // the global pipeline up to the one-sided viscous fluxes, then the records
  Epi ep;
  std::memset(&ep, 0, sizeof(ep));
  int rc = mx_residual(h->C, h->m, h->gr, q, nullptr, 0.0, ep, h->qtr, h->fci, h->wh, h->grad, h->fvn, h->fcv,
                       nullptr, nullptr, nullptr, S(stream));
  if (rc) return rc;
  int groups = 0;
  for (int p = 0; p < 6; ++p) groups += h->gr.cnt[p] ? 1 : 0;
  g_launches += groups * (h->m.kind == K_NS ? 2 : 1) + 2;
  return mx_records(h->C, h->m, h->qtr, h->fvn, rq, rw, rf, S(stream));
}

PMGB_API int pmgb_mdisc_element_residual(pmgb_mdisc* h, int32_t p, const int64_t* elems, int64_t B,
                                         const double* Q, const double* rq, const double* rw, const double* rf,
                                         double* out, void* stream) {
  if (!h || p < 0 || p > 5 || (B > 0 && (!elems || !Q || !rq || !out))) return -1;
  g_launches += 1;
  return mx_local(h->C, h->m, p, elems, B, Q, rq, rw, rf, out, S(stream));
}

PMGB_API int pmgb_disc_residual_path(pmgb_disc* h, int32_t want) {
  if (!h) return -1;
  // 0 general, 1 rectangle kernels (the faster chain per degree), 2 the four-kernel
  // chain, 3 the two-kernel chain (2, 3: A/B runs and cross-checks)
  if (want >= 0) h->d.has_rect = (want != 0 && h->d.rect.frec != nullptr) ? (want == 2 || want == 3 ? want : 1) : 0;
  return h->d.has_rect;
}

static int n_res_launches(const DiscDev& d) { return (d.kind == K_NS || d.kind == K_ADVD) ? 3 : 2; }

PMGB_API int pmgb_eval(pmgb_disc* h, const double* q, const double* X, double eps, const pmgb_epilogue* e,
                       double* out, void* stream) {
  if (!h || !q || !out || !e) return -1;
  Epi ep;
  ep.mode = e->mode;
  ep.s = e->s;
  ep.eps = e->eps;
  ep.adt = e->adt;
  ep.dtau = e->dtau;
  ep.sb_scalar = e->sb_scalar;
  ep.se_scalar = e->se_scalar;
  ep.X = e->X;
  ep.R0 = e->R0;
  ep.E = e->E;
  ep.Sb = e->Sb;
  ep.Se = e->Se;
  ep.Q0 = e->Q0;
  ep.dtau_e = e->dtau_e;
  ep.alpha = e->alpha;
  ep.npe = (int)((h->d.p + 1) * (h->d.p + 1) * h->d.nv);
  if (ep.mode == EPI_RK && (!ep.Q0 || !ep.dtau_e)) return -1;
  const bool rect = h->d.has_rect && rect_supported(h->d.p, h->d.kind);
  if (rect) {   // the rectangle kernels move whole points (4 doubles) per access
    const void* ps[] = {q, X, out, ep.X, ep.R0, ep.E, ep.Sb, ep.Se, ep.Q0};
    for (const void* p : ps)
      if (((uintptr_t)p & 31u) != 0) return -6;
  }
  g_launches += rect ? rect_launches(h->d, X != nullptr) : n_res_launches(h->d);
  return launch_residual(h->d, q, X, eps, ep, out, S(stream));
}

PMGB_API int pmgb_residual(pmgb_disc* h, const double* q, double* R, void* stream) {
  pmgb_epilogue e;
  std::memset(&e, 0, sizeof(e));
  e.mode = PMGB_EPI_R;
  return pmgb_eval(h, q, nullptr, 0.0, &e, R, stream);
}

PMGB_API int pmgb_jfnk_matvec(pmgb_disc* h, const double* X, const double* q, const double* R0, double shift,
                              double eps, double* out, void* stream) {
  pmgb_epilogue e;
  std::memset(&e, 0, sizeof(e));
  e.mode = PMGB_EPI_JV;
  e.s = shift;
  e.eps = eps;
  e.X = X;
  e.R0 = R0;
  return pmgb_eval(h, q, X, eps, &e, out, stream);
}

PMGB_API int pmgb_rk_lambda(pmgb_disc* h, const double* q, double adv_coef, double* lam, void* stream) {
  if (!h || (h->d.M > 0 && (!q || !lam)) || !(adv_coef > 0.0)) return -1;
  g_launches += 1;
  return launch_rk_lambda(h->d, q, adv_coef, lam, S(stream));
}

PMGB_API int pmgb_rk_dtau(int64_t M, const double* lam, double s, double cfl, double* dtau, void* stream) {
  if (M > 0 && (!lam || !dtau)) return -1;
  g_launches += 1;
  return launch_rk_dtau(M, lam, s, cfl, dtau, S(stream));
}

PMGB_API int pmgb_freeze(pmgb_disc* h, const double* q, double* qtr, double* fvn, void* stream) {
  if (!h || !q || !qtr) return -1;
  g_launches += n_res_launches(h->d) - 1;
  return launch_freeze(h->d, q, qtr, fvn, S(stream));
}

PMGB_API int pmgb_element_residual(pmgb_disc* h, const int64_t* elems, int64_t B, const double* Q,
                                   const double* qtr, const double* fvn, double* out, void* stream) {
  if (!h || (B > 0 && (!elems || !Q || !qtr || !out))) return -1;
  g_launches += 1;
  return launch_local_residual(h->d, elems, B, Q, qtr, fvn, out, S(stream));
}

PMGB_API int pmgb_blocks_invert(int64_t M, int32_t sz, const double* BT, double* XT, uint8_t* perm, void* stream) {
  if (!BT || !XT || !perm) return -1;
  g_launches += 1;
  return launch_inverse(M, sz, BT, XT, perm, S(stream), status_ptr());
}

PMGB_API int pmgb_blocks_assemble(pmgb_disc* h, const double* q, double shift, double eps, double* BT,
                                  double* XT, uint8_t* perm, void* stream) {
  if (!h || !q || !BT) return -1;
  const DiscDev& d = h->d;
  int rc = launch_freeze(d, q, d.qtr, d.fvn, S(stream));
  if (rc) return rc;
  rc = launch_blocks(d, q, d.qtr, d.fvn, shift, eps, BT, S(stream));
  if (rc) return rc;
  g_launches += n_res_launches(d);
  if (XT) {
    const int n = d.p + 1;
    return pmgb_blocks_invert(d.M, n * n * d.nv, BT, XT, perm, stream);
  }
  return 0;
}

PMGB_API int pmgb_sparse_assemble(pmgb_disc* h, const double* q, double shift, double eps, double* blocks,
                                  const int32_t* diag_slot, int64_t npairs, const int32_t* pair_e,
                                  const int8_t* pair_f, const int32_t* pair_slot, const int8_t* pair_add,
                                  const int64_t* wave_ptr, int32_t nwaves, void* stream) {
  if (!h || !q || !blocks || !diag_slot || nwaves < 0 || (npairs > 0 && (!pair_e || !pair_f || !pair_slot ||
                                                                         !pair_add || !wave_ptr)))
    return -1;
  const DiscDev& d = h->d;
  int rc = launch_freeze(d, q, d.qtr, d.fvn, S(stream));
  if (rc) return rc;
  rc = launch_blocks(d, q, d.qtr, d.fvn, shift, eps, blocks, S(stream), diag_slot);
  if (rc) return rc;
  g_launches += n_res_launches(d);
  for (int32_t w = 0; w < nwaves; ++w) {
    const int64_t b = wave_ptr[w], n = wave_ptr[w + 1] - wave_ptr[w];
    rc = launch_coupling(d, q, d.qtr, d.fvn, eps, n, pair_e + b, (const signed char*)pair_f + b, pair_slot + b,
                         (const signed char*)pair_add + b, blocks, S(stream));
    if (rc) return rc;
    g_launches += 1;
  }
  return 0;
}

PMGB_API int pmgb_sparse_matvec(int64_t n_rows, int32_t sz, const int32_t* indptr, const int32_t* indices,
                                const double* blocks, const double* x, double* y, void* stream) {
  if (!indptr || !indices || !blocks || !x || !y) return -1;
  g_launches += 1;
  return launch_sparse_matvec(n_rows, sz, indptr, indices, blocks, x, y, S(stream));
}

PMGB_API int pmgb_ilu0_factor(int64_t n_rows, int32_t sz, const int32_t* indptr, const int32_t* indices,
                               double* F, double* DX, uint8_t* DP, int32_t n_levels, const int64_t* level_ptr,
                               const int32_t* level_rows, const int32_t* level_diag, void* stream) {
  if (!indptr || !indices || !F || !DX || !DP || (n_levels > 0 && (!level_ptr || !level_rows || !level_diag)))
    return -1;
  (void)n_rows;
  for (int32_t L = 0; L < n_levels; ++L) {
    const int64_t b = level_ptr[L], n = level_ptr[L + 1] - level_ptr[L];
    int rc = launch_ilu_level(n, sz, level_rows + b, indptr, indices, F, DX, DP, S(stream));
    if (rc) return rc;
    rc = launch_inverse(n, sz, F, DX, DP, S(stream), status_ptr(), level_diag + b, level_rows + b, 4);
    if (rc) return rc;
    g_launches += 2;
  }
  return 0;
}

PMGB_API int pmgb_ilu0_apply(int64_t n_rows, int32_t sz, const int32_t* indptr, const int32_t* indices,
                              const double* F, const double* DX, const uint8_t* DP, int32_t n_lo,
                              const int64_t* lo_ptr, const int32_t* lo_rows, int32_t n_up, const int64_t* up_ptr,
                              const int32_t* up_rows, const double* x, double* y, double* out, void* stream) {
  if (!indptr || !indices || !F || !DX || !DP || !x || !y || !out) return -1;
  (void)n_rows;
  for (int32_t L = 0; L < n_lo; ++L) {
    const int64_t b = lo_ptr[L], n = lo_ptr[L + 1] - lo_ptr[L];
    int rc = launch_ilu_sweep(0, n, sz, lo_rows + b, indptr, indices, F, DX, DP, x, y, S(stream));
    if (rc) return rc;
  }
  for (int32_t L = 0; L < n_up; ++L) {
    const int64_t b = up_ptr[L], n = up_ptr[L + 1] - up_ptr[L];
    int rc = launch_ilu_sweep(1, n, sz, up_rows + b, indptr, indices, F, DX, DP, y, out, S(stream));
    if (rc) return rc;
  }
  g_launches += n_lo + n_up;
  return 0;
}

PMGB_API int pmgb_wall_forces(pmgb_disc* h, const double* q, int64_t n_wall, const int32_t* wall_e,
                              const int8_t* wall_f, const double* weights, double* out, void* stream) {
  if (!h || !q || !weights || (n_wall > 0 && (!wall_e || !wall_f || !out))) return -1;
  const DiscDev& d = h->d;
  if (d.kind != K_EULER && d.kind != K_NS) return -5;
  g_launches += (d.kind == K_NS) ? 3 : 2;
  return launch_forces(d, q, n_wall, wall_e, (const signed char*)wall_f, weights, out, S(stream));
}

PMGB_API int pmgb_ilu0_apply_fused(int32_t sz, const int32_t* row_entries, const double* F,
                                    const double* DX, const uint8_t* DP, int32_t n_lo, const int32_t* lo_ptr_dev,
                                    const int32_t* lo_rows, int32_t n_up, const int32_t* up_ptr_dev,
                                    const int32_t* up_rows, int32_t max_level_rows, const double* x, double* y,
                                    double* out, uint32_t* barrier, void* stream) {
  if (!row_entries || !F || !DX || !DP || !x || !y || !out || !barrier || !lo_ptr_dev || !up_ptr_dev)
    return -1;
  g_launches += 1;
  return launch_ilu_persistent(sz, n_lo, lo_ptr_dev, lo_rows, n_up, up_ptr_dev, up_rows, row_entries, F, DX,
                               DP, x, y, out, barrier, max_level_rows, S(stream));
}

PMGB_API int pmgb_ej_apply(int64_t M, int32_t sz, const double* XT, const uint8_t* perm, const double* x, double* y,
                           void* stream) {
  g_launches += 1;
  return launch_block_gemv(M, sz, XT, perm, x, 0.0, nullptr, y, S(stream));
}

PMGB_API int pmgb_ej_update(int64_t M, int32_t sz, const double* XT, const uint8_t* perm, const double* dd,
                            double omega, const double* base, double* out, void* stream) {
  if (!base) return -1;
  g_launches += 1;
  return launch_block_gemv(M, sz, XT, perm, dd, omega, base, out, S(stream));
}

PMGB_API int pmgb_blocks_demote(int64_t M, int32_t sz, const double* XT, float* XT32, void* stream) {
  if (M < 0 || sz <= 0 || (M > 0 && (!XT || !XT32))) return -1;
  g_launches += 1;
  return launch_demote(M * (int64_t)sz * sz, XT, XT32, S(stream));
}

PMGB_API int pmgb_ej_apply_f32(int64_t M, int32_t sz, const float* XT32, const uint8_t* perm, const double* x,
                               double* y, void* stream) {
  g_launches += 1;
  return launch_block_gemv_f32(M, sz, XT32, perm, x, 0.0, nullptr, y, S(stream));
}

PMGB_API int pmgb_ej_update_f32(int64_t M, int32_t sz, const float* XT32, const uint8_t* perm, const double* dd,
                                double omega, const double* base, double* out, void* stream) {
  if (!base) return -1;
  g_launches += 1;
  return launch_block_gemv_f32(M, sz, XT32, perm, dd, omega, base, out, S(stream));
}

PMGB_API int pmgb_transfer(int64_t M, int32_t nv, int32_t nin, int32_t nout, const double* T, const double* src,
                           const double* src_base, double* dst, int32_t accumulate, void* stream) {
  if (nin < 1 || nin > 6 || nout < 1 || nout > 6) return -1;
  g_launches += 1;
  return launch_transfer(M, nv, nin, nout, T, src, src_base, dst, accumulate, S(stream));
}

PMGB_API int pmgb_dot(int64_t n, const double* x, const double* y, double* r, void* stream) {
  g_launches += 1;
  return launch_dot(n, x, y, r, 0, S(stream));
}

PMGB_API int pmgb_nrm2(int64_t n, const double* x, double* r, void* stream) {
  g_launches += 1;
  return launch_dot(n, x, x, r, 1, S(stream));
}

PMGB_API int pmgb_mgs(int64_t n, double* V, int64_t ld, int32_t j, double* w, double* H, double thresh,
                      int32_t* finite_dev, void* stream) {
  g_launches += j + 3;
  return launch_mgs(n, V, ld, j, w, H, thresh, finite_dev, S(stream));
}

PMGB_API int pmgb_mgs_pass(int64_t n, double* w, const double* Vprev, const double* hprev, const double* Vnext,
                           double* out, int32_t first, int32_t* finite_dev, void* stream) {
  if (n < 0 || !w || !Vnext || !out || (Vprev && !hprev)) return -1;
  g_launches += 1;
  return launch_mgs_pass(n, w, Vprev, hprev, Vnext, out, first, finite_dev, S(stream));
}

PMGB_API int pmgb_multidot(int64_t n, const double* V, int64_t ld, int32_t k, const double* w, double* out_dev,
                           int32_t* finite_dev, void* stream) {
  if (n < 0 || !V || !w || !out_dev) return -1;
  g_launches += 1;
  return launch_multidot(n, V, ld, k, w, out_dev, finite_dev, S(stream));
}

PMGB_API int pmgb_gemv_sub(int64_t n, int32_t k, const double* V, int64_t ld, const double* y_dev, double* w,
                           void* stream) {
  if (n < 0 || !V || !y_dev || !w) return -1;
  g_launches += 1;
  return launch_gemv_sub(n, k, V, ld, y_dev, w, S(stream));
}

PMGB_API int pmgb_normalize_sqrt(int64_t n, const double* w, double* h_dev, double thresh, double* v,
                                 void* stream) {
  if (n < 0 || !w || !h_dev || !v) return -1;
  g_launches += 2;
  return launch_normalize_sqrt(n, w, h_dev, thresh, v, S(stream));
}

PMGB_API int pmgb_lincomb(int64_t n, int32_t k, const double* c, const double* const* xs, double* out,
                          void* stream) {
  g_launches += 1;
  return launch_lincomb(n, k, c, xs, out, S(stream));
}

PMGB_API int pmgb_gemv_t(int64_t n, int32_t k, const double* V, int64_t ld, const double* y, double* out,
                         void* stream) {
  g_launches += 1;
  return launch_gemv_t(n, k, V, ld, y, out, S(stream));
}

PMGB_API int pmgb_any_nonzero(int64_t n, const double* x, int32_t* flag, void* stream) {
  g_launches += 1;
  return launch_any_nonzero(n, x, flag, S(stream));
}

PMGB_API int pmgb_status(void* stream, int32_t* kind, int64_t* element, int32_t clear) {
  Status s;
  const int rc = status_read(S(stream), &s, clear);
  if (kind) *kind = s.kind;
  if (element) *element = s.element;
  return rc;
}

PMGB_API int pmgb_status_clear(void* stream) { return status_clear_async(S(stream)); }

PMGB_API int pmgb_sync(void* stream) { return (int)cudaStreamSynchronize(S(stream)); }

PMGB_API int pmgb_probe_fp64(int64_t iters, int32_t blocks, double* out_dev, void* stream) {
  return launch_probe_fp64(iters, blocks, out_dev, S(stream));
}

}  // extern "C"
