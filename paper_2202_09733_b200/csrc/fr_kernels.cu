// FR residual R(u), its fused Jv / defect epilogues, the frozen-neighbour
// element-local residual and the finite-difference element-Jacobi block
// assembly -- hand-written FP64 kernels for sm_100a.
//
// Reference behaviour (/root/reference/pkg/src/pmgflow/spatial.py):
//   residual 501-570  -> k_trace (phase 1) + k_fvn (phase 2) + k_assemble (phase 3)
//   freeze 700-766    -> k_trace + k_fvn into caller buffers (the frozen
//                        records are exactly the neighbours' traces / fvn)
//   element_residual 768-853 -> k_local (one fused kernel, own-side fluxes)
//   newton_krylov.py:174-201 (element_jacobian_block/assemble) -> k_blocks
//
// Thread mapping: one thread per solution point, EPB elements per CTA,
// face work strided over the same CTA; operators staged in shared memory.
// BR1 reaches two elements deep, so the global residual is split at the
// two neighbour exchanges (traces, then one-sided viscous fluxes).
#include <climits>
#include <cstdio>

#include "pmgb_internal.cuh"

namespace pmgb {

// ---------------------------------------------------------------------------
// shared-memory layout (in doubles) per CTA

template <int P, int KIND>
struct SL {
  using B = BC<P>;
  using T = KT<KIND>;
  static constexpr int E = B::EPB, N = B::N, NP = B::NP, NV = T::NV, NW = T::NW;
  static constexpr int OP = 0;                       // D(36) eL eR lL lR xg (6 each)
  static constexpr int Q = OP + 72;                  // [E][NP][NV]
  static constexpr int G = Q + E * NP * NV;          // [E][20]
  static constexpr int W = G + E * 20;               // [E][NP][NW]
  static constexpr int FC = W + E * NP * NW;         // [E][4][N][NV]  common face flux, CCW
  static constexpr int WH = FC + E * 4 * N * NV;     // [E][4][N][NW]  BR1 common value, CCW
  static constexpr int CG = WH + E * 4 * N * NW;     // [E][2][4][N][NW] gradient lifting terms (line idx)
  static constexpr int GR = CG + E * 8 * N * NW;     // [E][NP][2][NW] gradients
  static constexpr int FT = GR + E * NP * 2 * NW;    // [E][NP][NV]
  static constexpr int GT = FT + E * NP * NV;        // [E][NP][NV]
  static constexpr int CF = GT + E * NP * NV;        // [E][4][N][NV]  flux lifting terms (line idx)
  static constexpr int TR = CF + E * 4 * N * NV;     // [E][4][N][NV]  own traces, CCW
  static constexpr int R0 = TR + E * 4 * N * NV;     // [NP*NV] unperturbed local residual (blocks)
  static constexpr int TOTAL = R0 + NP * NV;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
};

struct Ops {
  const double* D;
  const double* eL;
  const double* eR;
  const double* lL;
  const double* lR;
  const double* xg;
};

__device__ __forceinline__ Ops stage_ops(const FrConst& C, double* sm) {
  for (int i = threadIdx.x; i < 66; i += blockDim.x) {
    double v;
    if (i < 36) v = C.D[i];
    else if (i < 42) v = C.eL[i - 36];
    else if (i < 48) v = C.eR[i - 42];
    else if (i < 54) v = C.lL[i - 48];
    else if (i < 60) v = C.lR[i - 54];
    else v = C.xg[i - 60];
    sm[i] = v;
  }
  return Ops{sm, sm + 36, sm + 42, sm + 48, sm + 54, sm + 60};
}

// point on face f, face point k, interpolation-line position i
template <int N>
__device__ __forceinline__ int fpt(int f, int k, int i) {
  return f == 0 ? i * N + k : f == 1 ? k * N + i : f == 2 ? i * N + (N - 1 - k) : (N - 1 - k) * N + i;
}

// ---------------------------------------------------------------------------
// pointwise physics (spatial.py:94-203)

struct Phys {
  double gamma, mu, kappa, ax, ay, diff;
};

__device__ __forceinline__ void prim(const double* q, double g, double& r, double& u, double& v, double& p) {
  r = q[0];
  const double ir = 1.0 / r;
  u = q[1] * ir;
  v = q[2] * ir;
  p = (g - 1.0) * (q[3] - 0.5 * r * (u * u + v * v));
}

// Roe flux along (nx, ny), no entropy fix (spatial.py:113-163)
__device__ __forceinline__ void roe(const double* qL, const double* qR, double nx, double ny, double g,
                                    double* F) {
  double rL, uL, vL, pL, rR, uR, vR, pR;
  prim(qL, g, rL, uL, vL, pL);
  prim(qR, g, rR, uR, vR, pR);
  const double HL = (qL[3] + pL) / rL;
  const double HR = (qR[3] + pR) / rR;
  const double sL = sqrt(rL), sR = sqrt(rR);
  const double w = sL / (sL + sR), w1 = 1.0 - w;
  const double u = w * uL + w1 * uR;
  const double v = w * vL + w1 * vR;
  const double H = w * HL + w1 * HR;
  const double ke = 0.5 * (u * u + v * v);
  const double c2 = (g - 1.0) * (H - ke);
  const double c = sqrt(c2);
  const double rb = sL * sR;
  const double un = u * nx + v * ny;
  const double du = uR - uL, dv = vR - vL;
  const double dn = du * nx + dv * ny;
  const double dtg = -du * ny + dv * nx;
  const double dp = pR - pL;
  const double i2 = 1.0 / (2.0 * c2);
  const double k1 = fabs(un - c) * ((dp - rb * c * dn) * i2);
  const double k2 = fabs(un) * ((rR - rL) - dp / c2);
  const double k3 = fabs(un) * (rb * dtg);
  const double k4 = fabs(un + c) * ((dp + rb * c * dn) * i2);
  const double ut = -u * ny + v * nx;
  const double d0 = k1 + k2 + k4;
  const double d1 = k1 * (u - c * nx) + k2 * u - k3 * ny + k4 * (u + c * nx);
  const double d2 = k1 * (v - c * ny) + k2 * v + k3 * nx + k4 * (v + c * ny);
  const double d3 = k1 * (H - c * un) + k2 * ke + k3 * ut + k4 * (H + c * un);
  const double qnL = uL * nx + vL * ny, qnR = uR * nx + vR * ny;
  const double EpL = qL[3] + pL, EpR = qR[3] + pR;
  F[0] = 0.5 * (qL[0] * qnL + qR[0] * qnR) - 0.5 * d0;
  F[1] = 0.5 * ((qL[1] * qnL + pL * nx) + (qR[1] * qnR + pR * nx)) - 0.5 * d1;
  F[2] = 0.5 * ((qL[2] * qnL + pL * ny) + (qR[2] * qnR + pR * ny)) - 0.5 * d2;
  F[3] = 0.5 * (EpL * qnL + EpR * qnR) - 0.5 * d3;
}

template <int KIND>
__device__ __forceinline__ void num_flux(const double* qa, const double* qc, double nx, double ny,
                                         const Phys& ph, double* F) {
  if constexpr (KT<KIND>::FLOW) {
    roe(qa, qc, nx, ny, ph.gamma, F);
  } else {
    const double an = ph.ax * nx + ph.ay * ny;
    F[0] = 0.5 * an * (qa[0] + qc[0]) - 0.5 * fabs(an) * (qc[0] - qa[0]);
  }
}

template <int KIND>
__device__ __forceinline__ void ghost(const double* q, int tag, double nx, double ny, const double* qinf,
                                      double* gq) {
  if constexpr (KT<KIND>::FLOW) {
    if (tag == T_FAR_FIELD) {
      for (int v = 0; v < 4; ++v) gq[v] = qinf[v];
    } else if (tag == T_WALL_SLIP) {
      const double un = q[1] * nx + q[2] * ny;
      gq[0] = q[0];
      gq[1] = q[1] - 2.0 * un * nx;
      gq[2] = q[2] - 2.0 * un * ny;
      gq[3] = q[3];
    } else {
      gq[0] = q[0];
      gq[1] = -q[1];
      gq[2] = -q[2];
      gq[3] = q[3];
    }
  } else {
    gq[0] = (tag == T_FAR_FIELD) ? 0.0 : q[0];
  }
}

// viscous variables W (spatial.py:448-454)
template <int KIND>
__device__ __forceinline__ void grad_vars(const double* q, double g, double* w) {
  if constexpr (KT<KIND>::FLOW) {
    const double r = q[0], ir = 1.0 / r;
    const double u = q[1] * ir, v = q[2] * ir;
    const double p = (g - 1.0) * (q[3] - 0.5 * r * (u * u + v * v));
    w[0] = u;
    w[1] = v;
    w[2] = p * ir;
  } else {
    w[0] = q[0];
  }
}

// viscous flux vectors (spatial.py:166-180) -- ADVD: k grad
template <int KIND>
__device__ __forceinline__ void visc_flux(const double* q, const double* gx, const double* gy, const Phys& ph,
                                          double* fx, double* fy) {
  if constexpr (KT<KIND>::FLOW) {
    const double ir = 1.0 / q[0];
    const double u = q[1] * ir, v = q[2] * ir;
    const double d = gx[0] + gy[1];
    const double txx = ph.mu * (2.0 * gx[0] - (2.0 / 3.0) * d);
    const double tyy = ph.mu * (2.0 * gy[1] - (2.0 / 3.0) * d);
    const double txy = ph.mu * (gy[0] + gx[1]);
    fx[0] = 0.0;
    fx[1] = txx;
    fx[2] = txy;
    fx[3] = u * txx + v * txy + ph.kappa * gx[2];
    fy[0] = 0.0;
    fy[1] = txy;
    fy[2] = tyy;
    fy[3] = u * txy + v * tyy + ph.kappa * gy[2];
  } else {
    fx[0] = ph.diff * gx[0];
    fy[0] = ph.diff * gy[0];
  }
}

template <int KIND>
__device__ __forceinline__ void inv_flux(const double* q, const Phys& ph, double* fx, double* fy) {
  if constexpr (KT<KIND>::FLOW) {
    double r, u, v, p;
    prim(q, ph.gamma, r, u, v, p);
    fx[0] = q[1];
    fx[1] = q[1] * u + p;
    fx[2] = q[1] * v;
    fx[3] = u * (q[3] + p);
    fy[0] = q[2];
    fy[1] = q[2] * u;
    fy[2] = q[2] * v + p;
    fy[3] = v * (q[3] + p);
  } else {
    fx[0] = ph.ax * q[0];
    fy[0] = ph.ay * q[0];
  }
}

__device__ __forceinline__ bool physical(const double* q, double g) {
  double r, u, v, p;
  prim(q, g, r, u, v, p);
  return (r > 0.0) && (p > 0.0);
}

// bilinear metrics from the packed geometry record (mesh.pack_geometry)
struct Metric {
  double a0, a1, b0, b1, c0, c1, d0, d1;
  __device__ __forceinline__ double J00(double eta) const { return a0 + a1 * eta; }  // x_xi
  __device__ __forceinline__ double J10(double eta) const { return b0 + b1 * eta; }  // y_xi
  __device__ __forceinline__ double J01(double xi) const { return c0 + c1 * xi; }    // x_eta
  __device__ __forceinline__ double J11(double xi) const { return d0 + d1 * xi; }    // y_eta
};
__device__ __forceinline__ Metric metric(const double* g) {
  return Metric{g[0], g[1], g[2], g[3], g[4], g[5], g[6], g[7]};
}

__device__ __forceinline__ Phys phys_of(const FrConst& C) {
  return Phys{C.gamma, C.mu, C.kappa, C.adv_x, C.adv_y, C.diff};
}

// ---------------------------------------------------------------------------
// staging helpers

template <int P, int NV>
__device__ __forceinline__ void load_points(const double* __restrict__ src, int64_t e0, int64_t M, double* sQ) {
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB;
  const int64_t nval = (int64_t)E * NP * NV;
  const int64_t lim = (M - e0) * NP * NV;
  const double* base = src + e0 * NP * NV;
  for (int i = threadIdx.x; i < nval; i += blockDim.x) sQ[i] = (i < lim) ? __ldg(base + i) : 1.0;
}

template <int P>
__device__ __forceinline__ void load_geom(const double* __restrict__ geom, int64_t e0, int64_t M, double* sG) {
  constexpr int E = BC<P>::EPB;
  const int64_t lim = (M - e0) * 20;
  const double* base = geom + e0 * 20;
  for (int i = threadIdx.x; i < E * 20; i += blockDim.x) sG[i] = (i < lim) ? __ldg(base + i) : 0.0;
}

// trace of smem point array X[NP][C] component c at face (f, k)
template <int N, int C>
__device__ __forceinline__ double line_sum(const Ops& op, const double* X, int f, int k, int c) {
  const double* w = (f == 0 || f == 3) ? op.eL : op.eR;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) s += w[i] * X[fpt<N>(f, k, i) * C + c];
  return s;
}

// ---------------------------------------------------------------------------
// BR1 gradient pieces (spatial.py:594-603 via _divergence 407-430)

// face thread: lifting terms for the x and y gradients at (f, k) -> line index j
template <int P, int KIND>
__device__ __forceinline__ void grad_corrections(const Ops& op, const double* sW, const double* sG_el,
                                                 const double* sWH_el, double* sCG_el, int f, int k) {
  constexpr int N = P + 1, NW = KT<KIND>::NW;
  const Metric mt = metric(sG_el);
  const double nx = sG_el[8 + 2 * f], ny = sG_el[9 + 2 * f], js = sG_el[16 + f];
  const double sgn = (f == 1 || f == 2) ? 1.0 : -1.0;
  const int j = (f >= 2) ? N - 1 - k : k;
  const bool xiline = (f == 1 || f == 3);
  const double* w = (f == 0 || f == 3) ? op.eL : op.eR;
  double lx[NW], ly[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c) lx[c] = ly[c] = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double x = op.xg[i];
    // x-gradient: Ft = J11 W (xi lines), Gt = -J10 W (eta lines)
    // y-gradient: Ft = -J01 W,           Gt =  J00 W
    const double fxx = xiline ? mt.J11(x) : -mt.J10(x);
    const double fyy = xiline ? -mt.J01(x) : mt.J00(x);
    const double* Wp = sW + fpt<N>(f, k, i) * NW;
#pragma unroll
    for (int c = 0; c < NW; ++c) {
      lx[c] += w[i] * (fxx * Wp[c]);
      ly[c] += w[i] * (fyy * Wp[c]);
    }
  }
  const double* wh = sWH_el + (f * N + k) * NW;
#pragma unroll
  for (int c = 0; c < NW; ++c) {
    sCG_el[((0 * 4 + f) * N + j) * NW + c] = sgn * js * (nx * wh[c]) - lx[c];
    sCG_el[((1 * 4 + f) * N + j) * NW + c] = sgn * js * (ny * wh[c]) - ly[c];
  }
}

// point thread: corrected gradients at (a, b)
template <int P, int KIND>
__device__ __forceinline__ void gradient_at(const Ops& op, const double* sW, const double* sG_el,
                                            const double* sCG_el, int a, int b, double* gx, double* gy) {
  constexpr int N = P + 1, NW = KT<KIND>::NW;
  const Metric mt = metric(sG_el);
  double sx[NW], sy[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c) sx[c] = sy[c] = 0.0;
  // d/dxi of Ft along row a, d/deta of Gt along column b
  double dx[NW], dy[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c) dx[c] = dy[c] = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double Db = op.D[b * N + i], Da = op.D[a * N + i];
    const double xi = op.xg[i];
    const double* Wr = sW + (a * N + i) * NW;  // row a, column i
    const double* Wc = sW + (i * N + b) * NW;  // row i, column b
    const double j11 = mt.J11(xi), j01 = mt.J01(xi);   // xi_i dependence (row line)
    const double j10 = mt.J10(xi), j00 = mt.J00(xi);   // eta_i dependence (column line)
#pragma unroll
    for (int c = 0; c < NW; ++c) {
      sx[c] += Db * (j11 * Wr[c]);
      sy[c] += Db * (-j01 * Wr[c]);
      dx[c] += Da * (-j10 * Wc[c]);
      dy[c] += Da * (j00 * Wc[c]);
    }
  }
  const double xa = op.xg[a], xb = op.xg[b];
  const double det = mt.J00(xa) * mt.J11(xb) - mt.J01(xb) * mt.J10(xa);
  const double* cx = sCG_el;
  const double* cy = sCG_el + 4 * N * NW;
#pragma unroll
  for (int c = 0; c < NW; ++c) {
    double vx = sx[c] + dx[c];
    vx = vx + op.lR[b] * cx[(1 * N + a) * NW + c];
    vx = vx - op.lL[b] * cx[(3 * N + a) * NW + c];
    vx = vx + op.lR[a] * cx[(2 * N + b) * NW + c];
    vx = vx - op.lL[a] * cx[(0 * N + b) * NW + c];
    double vy = sy[c] + dy[c];
    vy = vy + op.lR[b] * cy[(1 * N + a) * NW + c];
    vy = vy - op.lL[b] * cy[(3 * N + a) * NW + c];
    vy = vy + op.lR[a] * cy[(2 * N + b) * NW + c];
    vy = vy - op.lL[a] * cy[(0 * N + b) * NW + c];
    gx[c] = vx / det;
    gy[c] = vy / det;
  }
}

// point thread: total flux (inviscid - viscous), transformed -> sFT/sGT
template <int P, int KIND>
__device__ __forceinline__ void point_fluxes(const double* q, const double* gx, const double* gy,
                                             const Phys& ph, const Metric& mt, double xa, double xb,
                                             double* Ft, double* Gt) {
  constexpr int NV = KT<KIND>::NV;
  double fx[NV], fy[NV];
  inv_flux<KIND>(q, ph, fx, fy);
  if constexpr (KT<KIND>::VISC) {
    double vx[NV], vy[NV];
    visc_flux<KIND>(q, gx, gy, ph, vx, vy);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      fx[v] = fx[v] - vx[v];
      fy[v] = fy[v] - vy[v];
    }
  }
  const double j00 = mt.J00(xa), j10 = mt.J10(xa), j01 = mt.J01(xb), j11 = mt.J11(xb);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    Ft[v] = j11 * fx[v] - j01 * fy[v];
    Gt[v] = -j10 * fx[v] + j00 * fy[v];
  }
}

// face thread: FR lifting term of the flux divergence, line index j
template <int P, int KIND>
__device__ __forceinline__ void flux_corrections(const Ops& op, const double* sFT_el, const double* sGT_el,
                                                 const double* sG_el, const double* Fc, double* sCF_el,
                                                 int f, int k) {
  constexpr int N = P + 1, NV = KT<KIND>::NV;
  const double js = sG_el[16 + f];
  const double sgn = (f == 1 || f == 2) ? 1.0 : -1.0;
  const int j = (f >= 2) ? N - 1 - k : k;
  const double* X = (f == 1 || f == 3) ? sFT_el : sGT_el;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double l = line_sum<N, NV>(op, X, f, k, v);
    sCF_el[(f * N + j) * NV + v] = sgn * js * Fc[v] - l;
  }
}

// point thread: -div / det (spatial.py:407-430, 627)
template <int P, int KIND>
__device__ __forceinline__ void divergence_at(const Ops& op, const double* sFT_el, const double* sGT_el,
                                              const double* sCF_el, const Metric& mt, int a, int b,
                                              double* R) {
  constexpr int N = P + 1, NV = KT<KIND>::NV;
  double s[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) s[v] = 0.0;
  double t[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) t[v] = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double Db = op.D[b * N + i], Da = op.D[a * N + i];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      s[v] += Db * sFT_el[(a * N + i) * NV + v];
      t[v] += Da * sGT_el[(i * N + b) * NV + v];
    }
  }
  const double xa = op.xg[a], xb = op.xg[b];
  const double det = mt.J00(xa) * mt.J11(xb) - mt.J01(xb) * mt.J10(xa);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double d = s[v] + t[v];
    d = d + op.lR[b] * sCF_el[(1 * N + a) * NV + v];
    d = d - op.lL[b] * sCF_el[(3 * N + a) * NV + v];
    d = d + op.lR[a] * sCF_el[(2 * N + b) * NV + v];
    d = d - op.lL[a] * sCF_el[(0 * N + b) * NV + v];
    R[v] = -(d / det);
  }
}

// ---------------------------------------------------------------------------
// phase 1: traces (+ optional q + eps X prologue, + physicality flags)

template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS)
k_trace(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ X,
        double eps, double* __restrict__ qp, double* __restrict__ qtr, int* __restrict__ bad) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB, NV = KT<KIND>::NV;
  const Ops op = stage_ops(C, sm);
  double* sQ = sm + L::Q;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int64_t M = m.M;
  if (X == nullptr) {
    load_points<P, NV>(q, e0, M, sQ);
  } else {
    // q + eps * X, rounded as the reference does (newton_krylov.py:76)
    const int64_t nval = (int64_t)E * NP * NV, lim = (M - e0) * NP * NV;
    const double* qb = q + e0 * NP * NV;
    const double* xb = X + e0 * NP * NV;
    double* pb = qp + e0 * NP * NV;
    for (int i = threadIdx.x; i < nval; i += blockDim.x) {
      double v = 1.0;
      if (i < lim) {
        v = __dadd_rn(__ldg(qb + i), __dmul_rn(eps, __ldg(xb + i)));
        pb[i] = v;
      }
      sQ[i] = v;
    }
  }
  __syncthreads();
  const double g = C.gamma;
  if constexpr (KT<KIND>::FLOW) {
    if (bad != nullptr) {
      const int t = threadIdx.x;
      if (t < E * NP) {
        const int64_t e = e0 + t / NP;
        if (e < M && !physical(sQ + t * NV, g)) atomicMin(bad, (int)e);
      }
    }
  }
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = e0 + el;
    if (e >= M) continue;
    const double* Qe = sQ + el * NP * NV;
    double tr[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = line_sum<N, NV>(op, Qe, f, k, v);
    if constexpr (KT<KIND>::FLOW) {
      if (bad != nullptr && !physical(tr, g)) atomicMin(bad + 1, (int)e);
    }
    double* dst = qtr + ((e * 4 + f) * N + k) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) dst[v] = tr[v];
  }
}

// ---------------------------------------------------------------------------
// phase 2: one-sided viscous normal flux on every face (spatial.py:536-557)

template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS)
k_fvn(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
      double* __restrict__ fvn) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW;
  const Ops op = stage_ops(C, sm);
  double* sQ = sm + L::Q;
  double* sG = sm + L::G;
  double* sW = sm + L::W;
  double* sWH = sm + L::WH;
  double* sCG = sm + L::CG;
  double* sGR = sm + L::GR;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int64_t M = m.M;
  const Phys ph = phys_of(C);
  load_points<P, NV>(q, e0, M, sQ);
  load_geom<P>(m.geom, e0, M, sG);
  __syncthreads();
  const int t0 = threadIdx.x;
  if (t0 < E * NP) grad_vars<KIND>(sQ + t0 * NV, ph.gamma, sW + t0 * NW);
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = e0 + el;
    if (e >= M) continue;
    const int2 lk = m.link[e * 4 + f];
    double tr[NV], nb[NV];
    const double* src = qtr + ((e * 4 + f) * N + k) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = __ldg(src + v);
    if (lk.x >= 0) {
      const int kk = lk_rev(lk.y) ? N - 1 - k : k;
      const double* ns = qtr + (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV;
#pragma unroll
      for (int v = 0; v < NV; ++v) nb[v] = __ldg(ns + v);
    } else {
      const double* gq = sG + el * 20;
      ghost<KIND>(tr, lk_tag(lk.y), gq[8 + 2 * f], gq[9 + 2 * f], C.qinf, nb);
    }
    double wa[NW], wc[NW];
    grad_vars<KIND>(tr, ph.gamma, wa);
    grad_vars<KIND>(nb, ph.gamma, wc);
    double* wh = sWH + ((el * 4 + f) * N + k) * NW;
#pragma unroll
    for (int c = 0; c < NW; ++c) wh[c] = 0.5 * (wa[c] + wc[c]);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    if (e0 + el >= M) continue;
    grad_corrections<P, KIND>(op, sW + el * NP * NW, sG + el * 20, sWH + el * 4 * N * NW,
                              sCG + el * 8 * N * NW, f, k);
  }
  __syncthreads();
  if (t0 < E * NP) {
    const int el = t0 / NP, pt = t0 % NP;
    double gx[NW], gy[NW];
    gradient_at<P, KIND>(op, sW + el * NP * NW, sG + el * 20, sCG + el * 8 * N * NW, pt / N, pt % N, gx, gy);
#pragma unroll
    for (int c = 0; c < NW; ++c) {
      sGR[(t0 * 2 + 0) * NW + c] = gx[c];
      sGR[(t0 * 2 + 1) * NW + c] = gy[c];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = e0 + el;
    if (e >= M) continue;
    const double* GRe = sGR + el * NP * 2 * NW;
    double gx[NW], gy[NW];
#pragma unroll
    for (int c = 0; c < NW; ++c) {
      gx[c] = line_sum<N, 2 * NW>(op, GRe, f, k, c);
      gy[c] = line_sum<N, 2 * NW>(op, GRe, f, k, NW + c);
    }
    double tr[NV];
    const double* src = qtr + ((e * 4 + f) * N + k) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = __ldg(src + v);
    double fx[NV], fy[NV];
    visc_flux<KIND>(tr, gx, gy, ph, fx, fy);
    const double nx = sG[el * 20 + 8 + 2 * f], ny = sG[el * 20 + 9 + 2 * f];
    double* dst = fvn + ((e * 4 + f) * N + k) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) dst[v] = fx[v] * nx + fy[v] * ny;
  }
}

// ---------------------------------------------------------------------------
// phase 3: common fluxes, volume fluxes, FR divergence, fused epilogue

__device__ __forceinline__ double epi_apply(const Epi& ep, int64_t i, double R, double qv) {
  switch (ep.mode) {
    case EPI_R:
      return R;
    case EPI_F:
      return ep.s * qv - R;
    case EPI_DEFECT: {
      const double sb = ep.Sb ? ep.Sb[i] : ep.sb_scalar;
      const double se = ep.Se ? ep.Se[i] : ep.se_scalar;
      return (sb - (ep.s * qv - R)) + se;
    }
    case EPI_JV:
      return __dsub_rn(__dmul_rn(ep.s, ep.X[i]), __ddiv_rn(__dsub_rn(R, ep.R0[i]), ep.eps));
    case EPI_STAGE_F:
      return __dsub_rn(__ddiv_rn(__dsub_rn(qv, ep.E[i]), ep.adt), R);
    case EPI_STAGE_JV: {
      const double F = __dsub_rn(__ddiv_rn(__dsub_rn(qv, ep.E[i]), ep.adt), R);
      return __dadd_rn(__ddiv_rn(ep.X[i], ep.dtau), __ddiv_rn(__dsub_rn(F, ep.R0[i]), ep.eps));
    }
    case EPI_NEG_R:
      return -R;
    case EPI_OUTER_F: {
      const double se = ep.Se ? ep.Se[i] : ep.se_scalar;
      return (ep.s * qv - R) - se;
    }
  }
  return R;
}

__device__ __forceinline__ void commit_status(int* bad, Status* st) {
  if (bad == nullptr) return;
  const int bs = bad[0], bt = bad[1];
  if (bs != INT_MAX || bt != INT_MAX) {
    if (st->kind == 0) {
      st->kind = (bs != INT_MAX) ? 1 : 2;
      st->element = (bs != INT_MAX) ? bs : bt;
    }
    bad[0] = INT_MAX;
    bad[1] = INT_MAX;
  }
}

template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS)
k_assemble(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
           const double* __restrict__ fvn, const Epi ep, double* __restrict__ out, int* bad, Status* st) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW;
  constexpr bool VISC = KT<KIND>::VISC;
  if (blockIdx.x == 0 && threadIdx.x == 0) commit_status(bad, st);
  const Ops op = stage_ops(C, sm);
  double* sQ = sm + L::Q;
  double* sG = sm + L::G;
  double* sW = sm + L::W;
  double* sFC = sm + L::FC;
  double* sWH = sm + L::WH;
  double* sCG = sm + L::CG;
  double* sFT = sm + L::FT;
  double* sGT = sm + L::GT;
  double* sCF = sm + L::CF;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int64_t M = m.M;
  const Phys ph = phys_of(C);
  load_points<P, NV>(q, e0, M, sQ);
  load_geom<P>(m.geom, e0, M, sG);
  __syncthreads();
  const int t0 = threadIdx.x;
  if constexpr (VISC) {
    if (t0 < E * NP) grad_vars<KIND>(sQ + t0 * NV, ph.gamma, sW + t0 * NW);
  }
  // common face fluxes: inviscid on the L side's normal (-F to R), viscous
  // 0.5 (fvn_own - fvn_nb), BR1 average (spatial.py:520-568)
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = e0 + el;
    if (e >= M) continue;
    const int2 lk = m.link[e * 4 + f];
    const double* gq = sG + el * 20;
    const double nx = gq[8 + 2 * f], ny = gq[9 + 2 * f];
    double tr[NV], nb[NV], F[NV];
    const int64_t own = ((e * 4 + f) * N + k) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = __ldg(qtr + own + v);
    int64_t nbi = -1;
    if (lk.x >= 0) {
      const int kk = lk_rev(lk.y) ? N - 1 - k : k;
      nbi = (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV;
#pragma unroll
      for (int v = 0; v < NV; ++v) nb[v] = __ldg(qtr + nbi + v);
      if (lk_left(lk.y)) {
        num_flux<KIND>(tr, nb, nx, ny, ph, F);
      } else {
        const double* gn = m.geom + (int64_t)lk.x * 20 + 8 + 2 * lk_face(lk.y);
        num_flux<KIND>(nb, tr, __ldg(gn), __ldg(gn + 1), ph, F);
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] = -F[v];
      }
    } else {
      ghost<KIND>(tr, lk_tag(lk.y), nx, ny, C.qinf, nb);
      num_flux<KIND>(tr, nb, nx, ny, ph, F);
    }
    if constexpr (VISC) {
      double wa[NW], wc[NW];
      grad_vars<KIND>(tr, ph.gamma, wa);
      grad_vars<KIND>(nb, ph.gamma, wc);
      double* wh = sWH + ((el * 4 + f) * N + k) * NW;
#pragma unroll
      for (int c = 0; c < NW; ++c) wh[c] = 0.5 * (wa[c] + wc[c]);
      double Fv[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) Fv[v] = __ldg(fvn + own + v);
      if (nbi >= 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) Fv[v] = 0.5 * (Fv[v] - __ldg(fvn + nbi + v));
      } else if (KT<KIND>::FLOW && lk_tag(lk.y) == T_WALL_ADIABATIC) {
        Fv[NV - 1] = 0.0;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) F[v] = F[v] - Fv[v];
    }
    double* fc = sFC + ((el * 4 + f) * N + k) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) fc[v] = F[v];
  }
  __syncthreads();
  if constexpr (VISC) {
    for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
      const int el = t / NF, r = t % NF, f = r / N, k = r % N;
      if (e0 + el >= M) continue;
      grad_corrections<P, KIND>(op, sW + el * NP * NW, sG + el * 20, sWH + el * 4 * N * NW,
                                sCG + el * 8 * N * NW, f, k);
    }
    __syncthreads();
  }
  if (t0 < E * NP) {
    const int el = t0 / NP, pt = t0 % NP, a = pt / N, b = pt % N;
    double gx[NW], gy[NW];
    if constexpr (VISC)
      gradient_at<P, KIND>(op, sW + el * NP * NW, sG + el * 20, sCG + el * 8 * N * NW, a, b, gx, gy);
    const Metric mt = metric(sG + el * 20);
    point_fluxes<P, KIND>(sQ + t0 * NV, gx, gy, ph, mt, op.xg[a], op.xg[b], sFT + t0 * NV, sGT + t0 * NV);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    if (e0 + el >= M) continue;
    flux_corrections<P, KIND>(op, sFT + el * NP * NV, sGT + el * NP * NV, sG + el * 20,
                              sFC + ((el * 4 + f) * N + k) * NV, sCF + el * 4 * N * NV, f, k);
  }
  __syncthreads();
  if (t0 < E * NP) {
    const int el = t0 / NP, pt = t0 % NP;
    const int64_t e = e0 + el;
    if (e < M) {
      const Metric mt = metric(sG + el * 20);
      double R[NV];
      divergence_at<P, KIND>(op, sFT + el * NP * NV, sGT + el * NP * NV, sCF + el * 4 * N * NV, mt,
                             pt / N, pt % N, R);
      const int64_t base = (e * NP + pt) * NV;
#pragma unroll
      for (int v = 0; v < NV; ++v) out[base + v] = epi_apply(ep, base + v, R[v], sQ[t0 * NV + v]);
    }
  }
}

// ---------------------------------------------------------------------------
// element-local residual with frozen neighbour data (spatial.py:768-853)
//
// Slot s of the CTA holds one (element, state) instance in sQ[s]; the
// neighbours enter only through the frozen traces qtr and one-sided
// viscous fluxes fvn of the linearisation state.  Fluxes are evaluated on
// the element's own normal (the reference's local path).  Leaves the
// local residual of point thread t in R (valid when t < E*NP and the
// slot is live).

template <int P, int KIND>
__device__ __forceinline__ void local_pipeline(const FrConst& C, const FrMesh& m, const Ops& op, double* sm,
                                               const int64_t* slot_elem, const double* __restrict__ qtr,
                                               const double* __restrict__ fvn, double* R) {
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW;
  constexpr bool VISC = KT<KIND>::VISC;
  double* sQ = sm + L::Q;
  double* sG = sm + L::G;
  double* sW = sm + L::W;
  double* sFC = sm + L::FC;
  double* sWH = sm + L::WH;
  double* sCG = sm + L::CG;
  double* sGR = sm + L::GR;
  double* sFT = sm + L::FT;
  double* sGT = sm + L::GT;
  double* sCF = sm + L::CF;
  double* sTR = sm + L::TR;
  const Phys ph = phys_of(C);
  const int t0 = threadIdx.x;
  if constexpr (VISC) {
    if (t0 < E * NP) grad_vars<KIND>(sQ + t0 * NV, ph.gamma, sW + t0 * NW);
  }
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = slot_elem[el];
    if (e < 0) continue;
    const int2 lk = m.link[e * 4 + f];
    const double* gq = sG + el * 20;
    const double nx = gq[8 + 2 * f], ny = gq[9 + 2 * f];
    const double* Qe = sQ + el * NP * NV;
    double tr[NV], nb[NV], F[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = line_sum<N, NV>(op, Qe, f, k, v);
    if (lk.x >= 0) {
      const int kk = lk_rev(lk.y) ? N - 1 - k : k;
      const double* ns = qtr + (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV;
#pragma unroll
      for (int v = 0; v < NV; ++v) nb[v] = __ldg(ns + v);
    } else {
      ghost<KIND>(tr, lk_tag(lk.y), nx, ny, C.qinf, nb);
    }
    num_flux<KIND>(tr, nb, nx, ny, ph, F);
    double* fc = sFC + ((el * 4 + f) * N + k) * NV;
    double* st = sTR + ((el * 4 + f) * N + k) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      fc[v] = F[v];
      st[v] = tr[v];
    }
    if constexpr (VISC) {
      double wa[NW], wc[NW];
      grad_vars<KIND>(tr, ph.gamma, wa);
      grad_vars<KIND>(nb, ph.gamma, wc);
      double* wh = sWH + ((el * 4 + f) * N + k) * NW;
#pragma unroll
      for (int c = 0; c < NW; ++c) wh[c] = 0.5 * (wa[c] + wc[c]);
    }
  }
  __syncthreads();
  if constexpr (VISC) {
    for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
      const int el = t / NF, r = t % NF, f = r / N, k = r % N;
      if (slot_elem[el] < 0) continue;
      grad_corrections<P, KIND>(op, sW + el * NP * NW, sG + el * 20, sWH + el * 4 * N * NW,
                                sCG + el * 8 * N * NW, f, k);
    }
    __syncthreads();
  }
  if (t0 < E * NP) {
    const int el = t0 / NP, pt = t0 % NP, a = pt / N, b = pt % N;
    double gx[NW], gy[NW];
    if constexpr (VISC) {
      gradient_at<P, KIND>(op, sW + el * NP * NW, sG + el * 20, sCG + el * 8 * N * NW, a, b, gx, gy);
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        sGR[(t0 * 2 + 0) * NW + c] = gx[c];
        sGR[(t0 * 2 + 1) * NW + c] = gy[c];
      }
    }
    const Metric mt = metric(sG + el * 20);
    point_fluxes<P, KIND>(sQ + t0 * NV, gx, gy, ph, mt, op.xg[a], op.xg[b], sFT + t0 * NV, sGT + t0 * NV);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < E * NF; t += blockDim.x) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = slot_elem[el];
    if (e < 0) continue;
    double* fc = sFC + ((el * 4 + f) * N + k) * NV;
    if constexpr (VISC) {
      const double* GRe = sGR + el * NP * 2 * NW;
      double gx[NW], gy[NW];
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        gx[c] = line_sum<N, 2 * NW>(op, GRe, f, k, c);
        gy[c] = line_sum<N, 2 * NW>(op, GRe, f, k, NW + c);
      }
      const double* tr = sTR + ((el * 4 + f) * N + k) * NV;
      double fx[NV], fy[NV];
      visc_flux<KIND>(tr, gx, gy, ph, fx, fy);
      const double nx = sG[el * 20 + 8 + 2 * f], ny = sG[el * 20 + 9 + 2 * f];
      const int2 lk = m.link[e * 4 + f];
      double Fv[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) Fv[v] = fx[v] * nx + fy[v] * ny;
      if (lk.x >= 0) {
        const int kk = lk_rev(lk.y) ? N - 1 - k : k;
        const double* ns = fvn + (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV;
#pragma unroll
        for (int v = 0; v < NV; ++v) Fv[v] = 0.5 * (Fv[v] + (-__ldg(ns + v)));
      } else if (KT<KIND>::FLOW && lk_tag(lk.y) == T_WALL_ADIABATIC) {
        Fv[NV - 1] = 0.0;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) fc[v] = fc[v] - Fv[v];
    }
    flux_corrections<P, KIND>(op, sFT + el * NP * NV, sGT + el * NP * NV, sG + el * 20, fc,
                              sCF + el * 4 * N * NV, f, k);
  }
  __syncthreads();
  if (t0 < E * NP) {
    const int el = t0 / NP, pt = t0 % NP;
    if (slot_elem[el] >= 0) {
      const Metric mt = metric(sG + el * 20);
      divergence_at<P, KIND>(op, sFT + el * NP * NV, sGT + el * NP * NV, sCF + el * 4 * N * NV, mt,
                             pt / N, pt % N, R);
    }
  }
}

// batched element-local residual: instance b = (elems[b], Q[b])
template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS)
k_local(const FrConst C, const FrMesh m, const int64_t* __restrict__ elems, int64_t B,
        const double* __restrict__ Q, const double* __restrict__ qtr, const double* __restrict__ fvn,
        double* __restrict__ out) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB, NV = KT<KIND>::NV;
  __shared__ int64_t slot[E];
  const Ops op = stage_ops(C, sm);
  const int64_t b0 = (int64_t)blockIdx.x * E;
  for (int s = threadIdx.x; s < E; s += blockDim.x) slot[s] = (b0 + s < B) ? elems[b0 + s] : -1;
  load_points<P, NV>(Q, b0, B, sm + L::Q);
  __syncthreads();
  for (int i = threadIdx.x; i < E * 20; i += blockDim.x) {
    const int64_t e = slot[i / 20];
    sm[L::G + i] = (e >= 0) ? __ldg(m.geom + e * 20 + i % 20) : 0.0;
  }
  __syncthreads();
  double R[NV];
  local_pipeline<P, KIND>(C, m, op, sm, slot, qtr, fvn, R);
  const int t0 = threadIdx.x;
  if (t0 < E * NP && b0 + t0 / NP < B) {
    double* dst = out + (b0 * NP + t0) * NV;
#pragma unroll
    for (int v = 0; v < NV; ++v) dst[v] = R[v];
  }
}

// FD element-Jacobi block: one CTA per element, columns in batches of EPB
// slots; column c perturbs local DoF c-1 by +eps (newton_krylov.py:174-184).
// Writes B^T (column-major block) so each column is a contiguous store.
template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS)
k_blocks(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
         const double* __restrict__ fvn, double shift, double eps, double* __restrict__ BT) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB, NV = KT<KIND>::NV;
  constexpr int SZ = NP * NV;
  __shared__ int64_t slot[E];
  const Ops op = stage_ops(C, sm);
  const int64_t e = blockIdx.x;
  double* sQ = sm + L::Q;
  double* sR0 = sm + L::R0;
  const double* qe = q + e * SZ;
  const int t0 = threadIdx.x;
  double* BTe = BT + e * (int64_t)SZ * SZ;
  for (int c0 = 0; c0 <= SZ; c0 += E) {
    __syncthreads();
    for (int s = threadIdx.x; s < E; s += blockDim.x) slot[s] = (c0 + s <= SZ) ? e : -1;
    for (int i = threadIdx.x; i < E * SZ; i += blockDim.x) {
      const int s = i / SZ, d = i % SZ, c = c0 + s;
      const double v = __ldg(qe + d);
      sQ[i] = (c >= 1 && d == c - 1) ? v + eps : v;
    }
    for (int i = threadIdx.x; i < E * 20; i += blockDim.x) sm[L::G + i] = __ldg(m.geom + e * 20 + i % 20);
    __syncthreads();
    double R[NV];
    local_pipeline<P, KIND>(C, m, op, sm, slot, qtr, fvn, R);
    const int s = t0 / NP, pt = t0 % NP, c = c0 + s;
    if (c0 == 0 && t0 < NP) {
#pragma unroll
      for (int v = 0; v < NV; ++v) sR0[pt * NV + v] = R[v];
    }
    __syncthreads();
    if (t0 < E * NP && c >= 1 && c <= SZ) {
      double* col = BTe + (int64_t)(c - 1) * SZ;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int i = pt * NV + v;
        double val = -(R[v] - sR0[i]) / eps;
        if (i == c - 1) val = val + shift;
        col[i] = val;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch

static __device__ int g_bad[2] = {INT_MAX, INT_MAX};
static __device__ Status g_status = {0, 0, 0};

template <int P, int KIND>
static int run_residual(const DiscDev& d, const double* q, const double* X, double eps, const Epi& epi,
                        double* out, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB, TH = BC<P>::THREADS;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trace<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k_fvn<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k_assemble<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    attr = true;
  }
  int* bad = nullptr;
  Status* stp = nullptr;
  cudaGetSymbolAddress((void**)&bad, g_bad);
  cudaGetSymbolAddress((void**)&stp, g_status);
  const unsigned grid = (unsigned)((d.M + E - 1) / E);
  const double* qq = q;
  if (X != nullptr) qq = d.qp;
  k_trace<P, KIND><<<grid, TH, L::BYTES, st>>>(d.C, d.mesh, q, X, eps, d.qp, d.qtr, bad);
  if (KT<KIND>::VISC) k_fvn<P, KIND><<<grid, TH, L::BYTES, st>>>(d.C, d.mesh, qq, d.qtr, d.fvn);
  k_assemble<P, KIND><<<grid, TH, L::BYTES, st>>>(d.C, d.mesh, qq, d.qtr, d.fvn, epi, out, bad, stp);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_freeze(const DiscDev& d, const double* q, double* qtr, double* fvn, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB, TH = BC<P>::THREADS;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trace<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k_fvn<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    attr = true;
  }
  const unsigned grid = (unsigned)((d.M + E - 1) / E);
  k_trace<P, KIND><<<grid, TH, L::BYTES, st>>>(d.C, d.mesh, q, nullptr, 0.0, nullptr, qtr, nullptr);
  if (KT<KIND>::VISC) k_fvn<P, KIND><<<grid, TH, L::BYTES, st>>>(d.C, d.mesh, q, qtr, fvn);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_local(const DiscDev& d, const int64_t* elems, int64_t B, const double* Q, const double* qtr,
                     const double* fvn, double* out, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB, TH = BC<P>::THREADS;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_local<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    attr = true;
  }
  if (B <= 0) return 0;
  const unsigned grid = (unsigned)((B + E - 1) / E);
  k_local<P, KIND><<<grid, TH, L::BYTES, st>>>(d.C, d.mesh, elems, B, Q, qtr, fvn, out);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_blocks(const DiscDev& d, const double* q, const double* qtr, const double* fvn, double shift,
                      double eps, double* BT, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int TH = BC<P>::THREADS;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_blocks<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    attr = true;
  }
  if (d.M <= 0) return 0;
  k_blocks<P, KIND><<<(unsigned)d.M, TH, L::BYTES, st>>>(d.C, d.mesh, q, qtr, fvn, shift, eps, BT);
  return (int)cudaGetLastError();
}

#define PMGB_DISPATCH(FN, ...)                                              \
  switch (d.kind * 8 + d.p) {                                               \
    case K_EULER * 8 + 0: return FN<0, K_EULER>(__VA_ARGS__);               \
    case K_EULER * 8 + 1: return FN<1, K_EULER>(__VA_ARGS__);               \
    case K_EULER * 8 + 2: return FN<2, K_EULER>(__VA_ARGS__);               \
    case K_EULER * 8 + 3: return FN<3, K_EULER>(__VA_ARGS__);               \
    case K_EULER * 8 + 4: return FN<4, K_EULER>(__VA_ARGS__);               \
    case K_EULER * 8 + 5: return FN<5, K_EULER>(__VA_ARGS__);               \
    case K_NS * 8 + 0: return FN<0, K_NS>(__VA_ARGS__);                     \
    case K_NS * 8 + 1: return FN<1, K_NS>(__VA_ARGS__);                     \
    case K_NS * 8 + 2: return FN<2, K_NS>(__VA_ARGS__);                     \
    case K_NS * 8 + 3: return FN<3, K_NS>(__VA_ARGS__);                     \
    case K_NS * 8 + 4: return FN<4, K_NS>(__VA_ARGS__);                     \
    case K_NS * 8 + 5: return FN<5, K_NS>(__VA_ARGS__);                     \
    case K_ADV * 8 + 0: return FN<0, K_ADV>(__VA_ARGS__);                   \
    case K_ADV * 8 + 1: return FN<1, K_ADV>(__VA_ARGS__);                   \
    case K_ADV * 8 + 2: return FN<2, K_ADV>(__VA_ARGS__);                   \
    case K_ADV * 8 + 3: return FN<3, K_ADV>(__VA_ARGS__);                   \
    case K_ADV * 8 + 4: return FN<4, K_ADV>(__VA_ARGS__);                   \
    case K_ADV * 8 + 5: return FN<5, K_ADV>(__VA_ARGS__);                   \
    case K_ADVD * 8 + 0: return FN<0, K_ADVD>(__VA_ARGS__);                 \
    case K_ADVD * 8 + 1: return FN<1, K_ADVD>(__VA_ARGS__);                 \
    case K_ADVD * 8 + 2: return FN<2, K_ADVD>(__VA_ARGS__);                 \
    case K_ADVD * 8 + 3: return FN<3, K_ADVD>(__VA_ARGS__);                 \
    case K_ADVD * 8 + 4: return FN<4, K_ADVD>(__VA_ARGS__);                 \
    case K_ADVD * 8 + 5: return FN<5, K_ADVD>(__VA_ARGS__);                 \
  }                                                                         \
  return -1000;

int launch_residual(const DiscDev& d, const double* q, const double* X, double eps, const Epi& epi,
                    double* out, cudaStream_t st) {
  PMGB_DISPATCH(run_residual, d, q, X, eps, epi, out, st)
}

int launch_freeze(const DiscDev& d, const double* q, double* qtr, double* fvn, cudaStream_t st) {
  PMGB_DISPATCH(run_freeze, d, q, qtr, fvn, st)
}

int launch_local_residual(const DiscDev& d, const int64_t* elems, int64_t B, const double* Q,
                          const double* qtr, const double* fvn, double* out, cudaStream_t st) {
  PMGB_DISPATCH(run_local, d, elems, B, Q, qtr, fvn, out, st)
}

int launch_blocks(const DiscDev& d, const double* q, const double* qtr, const double* fvn, double shift,
                  double eps, double* BT, cudaStream_t st) {
  PMGB_DISPATCH(run_blocks, d, q, qtr, fvn, shift, eps, BT, st)
}

Status* status_ptr() {
  Status* p = nullptr;
  cudaGetSymbolAddress((void**)&p, g_status);
  return p;
}

int status_clear_async(cudaStream_t st) {
  Status z = {0, 0, 0};
  int b[2] = {INT_MAX, INT_MAX};
  cudaMemcpyToSymbolAsync(g_status, &z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  cudaMemcpyToSymbolAsync(g_bad, b, sizeof(b), 0, cudaMemcpyHostToDevice, st);
  return (int)cudaStreamSynchronize(st);
}

int status_read(cudaStream_t st, Status* out, int clear) {
  cudaError_t e = cudaMemcpyFromSymbolAsync(out, g_status, sizeof(Status), 0, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return (int)e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return (int)e;
  if (clear && out->kind != 0) return status_clear_async(st);
  return 0;
}

}  // namespace pmgb
