// FR residual on MIXED-degree meshes (per-element degree map, p = 0..5):
// the reference's degree groups with mortar face transfers, for the
// p-adaptive path.
//
// Reference: /root/reference/pkg/src/pmgflow/spatial.py
//   residual 501-570 with _pair_align / _pair_scatter 468-497 and
//   _pair_scatter_values 572-585: on a face between degrees pL != pR both
//   sides' traces are interpolated (Pi) to the higher degree's face points,
//   the common flux / BR1 value is formed there and restricted (Gamma) back
//   to the lower side; the one-sided viscous fluxes likewise;
//   freeze 700-766 (neighbour records aligned and transferred to own
//   points: Pi from a lower neighbour, Gamma from a higher one);
//   element_residual 768-853.
//
// Data: the reference's flat layout (element e at offsets[e], (n_e, n_e, 4)
// C order); per element-face arrays padded to 6 points.  Kernels:
//   kmx_trace<P>  CTA per element of degree P: own face traces, checks
//   kmx_face      thread per face: mortar Roe flux + BR1 value (both sides)
//   kmx_grad<P>   CTA per element: BR1 gradients (general bilinear metric),
//                 stored; one-sided viscous fluxes on own faces
//   kmx_visc      thread per face: mortar common viscous flux
//   kmx_asm<P>    CTA per element: point fluxes, FR divergence, epilogue
//   kmx_records   thread per (element, face): frozen neighbour records
//   kmx_local<P>  CTA per (element, state): element-local residual
// One CTA per element keeps the code general (any bilinear element, any
// degree pairing); this path carries features, the uniform-degree paths
// carry the throughput.
#include <climits>

#include "fr_device.cuh"

namespace pmgb {

constexpr int MXN = 6;     // padded face points
constexpr int MXT = 64;    // threads per element CTA (>= 36 points, >= 24 face points)
constexpr int MX_OPS = 66; // per degree: D[36] eL eR lL lR xg [6 each]

struct MixDev {
  int64_t M;
  int kind;
  const int8_t* deg;      // (M)
  const int64_t* off;     // (M+1) doubles
  const int64_t* poff;    // (M+1) points (gradient scratch rows)
  const double* geom;     // (M,20)
  const int2* link;       // (M,4)
  const double* ops;      // (6, 66)
  const double* xfer;     // (6*6 pairs, 2, 6, 6): [pH][pL] Pi (nH x nL), Gamma (nL x nH)
  int64_t nface;
  const int4* faces;      // {eL, fL | rev<<2 | bnd<<3 | tag<<4, eR, fR}
};

__device__ __forceinline__ const double* xf_pi(const MixDev& m, int pH, int pL) {
  return m.xfer + ((pH * 6 + pL) * 2 + 0) * 36;
}
__device__ __forceinline__ const double* xf_gamma(const MixDev& m, int pH, int pL) {
  return m.xfer + ((pH * 6 + pL) * 2 + 1) * 36;
}

// per-element metric at every point (bilinear map; spatial.py via mesh.py:347-395)
template <int N>
struct ElemGeo {
  double j00[N * N], j10[N * N], j01[N * N], j11[N * N], det[N * N];
  double js[4];
};

template <int N>
__device__ __forceinline__ void load_ops(const MixDev& m, double* sops) {
  for (int i = threadIdx.x; i < MX_OPS; i += blockDim.x) sops[i] = m.ops[(N - 1) * MX_OPS + i];
}
#define MX_D(i, j) sops[(i) * N + (j)]
#define MX_EL(i) sops[36 + (i)]
#define MX_ER(i) sops[42 + (i)]
#define MX_LL(i) sops[48 + (i)]
#define MX_LR(i) sops[54 + (i)]
#define MX_XG(i) sops[60 + (i)]

template <int N>
__device__ __forceinline__ void load_geo(const double* g, const double* sops, ElemGeo<N>& G) {
  const Metric mt = metric(g);
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) {
    const double eta = MX_XG(t / N), xi = MX_XG(t % N);
    G.j00[t] = mt.J00(eta);
    G.j10[t] = mt.J10(eta);
    G.j01[t] = mt.J01(xi);
    G.j11[t] = mt.J11(xi);
    G.det[t] = G.j00[t] * G.j11[t] - G.j01[t] * G.j10[t];
  }
  if (threadIdx.x < 4) G.js[threadIdx.x] = g[16 + threadIdx.x];
}

// FR divergence of NV-variable contravariant fluxes Ft, Gt (point planes
// [v][N*N]) with normal face fluxes Fc ([f][k][v], own points, CCW), as
// spatial.py:407-430, divided by det; for point (a, b)
template <int N, int NV>
__device__ __forceinline__ void mx_div_at(const double* sops, const ElemGeo<N>& G, const double* Ft, const double* Gt,
                                          const double* Fc, int a, int b, double* out) {
  constexpr int NP = N * N;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double* ft = Ft + v * NP;
    const double* gt = Gt + v * NP;
    double s = 0.0, t2 = 0.0, ft1 = 0.0, ft3 = 0.0, gt2 = 0.0, gt0 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s += MX_D(b, i) * ft[a * N + i];
      t2 += MX_D(a, i) * gt[i * N + b];
      ft1 += MX_ER(i) * ft[a * N + i];
      ft3 += MX_EL(i) * ft[a * N + i];
      gt2 += MX_ER(i) * gt[i * N + b];
      gt0 += MX_EL(i) * gt[i * N + b];
    }
    double d = s + t2;
    const double fs1 = G.js[1] * Fc[(1 * MXN + a) * NV + v];
    const double fs3 = -G.js[3] * Fc[(3 * MXN + (N - 1 - a)) * NV + v];
    const double gs2 = G.js[2] * Fc[(2 * MXN + (N - 1 - b)) * NV + v];
    const double gs0 = -G.js[0] * Fc[(0 * MXN + b) * NV + v];
    d = d + MX_LR(b) * (fs1 - ft1);
    d = d - MX_LL(b) * (fs3 - ft3);
    d = d + MX_LR(a) * (gs2 - gt2);
    d = d - MX_LL(a) * (gs0 - gt0);
    out[v] = d / G.det[a * N + b];
  }
}

// BR1 gradients (spatial.py:594-603) of W (planes [3][NP]) with common
// values What ([f][k][3]) -> gx, gy planes; uses Ft/Gt scratch planes
template <int N>
__device__ __forceinline__ void mx_gradient(const double* sops, const ElemGeo<N>& G, const double* W,
                                            const double* What, const double* nrm, double* Ft, double* Gt,
                                            double* Fcs, double* gx, double* gy) {
  constexpr int NP = N * N;
  for (int comp = 0; comp < 2; ++comp) {
    // comp 0 (x): Ft = J11 W, Gt = -J10 W, Fc = nx What; comp 1 (y): Ft = -J01 W, Gt = J00 W, Fc = ny What
    for (int t = threadIdx.x; t < NP; t += blockDim.x)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double w = W[c * NP + t];
        Ft[c * NP + t] = comp == 0 ? G.j11[t] * w : -G.j01[t] * w;
        Gt[c * NP + t] = comp == 0 ? -G.j10[t] * w : G.j00[t] * w;
      }
    for (int t = threadIdx.x; t < 4 * MXN; t += blockDim.x) {
      const int f = t / MXN;
      const double nn = nrm[2 * f + comp];
#pragma unroll
      for (int c = 0; c < 3; ++c) Fcs[t * 3 + c] = nn * What[t * 3 + c];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < NP; t += blockDim.x) {
      double o[3];
      mx_div_at<N, 3>(sops, G, Ft, Gt, Fcs, t / N, t % N, o);
      double* dst = comp == 0 ? gx : gy;
#pragma unroll
      for (int c = 0; c < 3; ++c) dst[c * NP + t] = o[c];
    }
    __syncthreads();
  }
}

// traces of NV point planes on the 4 faces (CCW), as spatial.py:398-405
template <int N, int NV>
__device__ __forceinline__ void mx_traces(const double* sops, const double* X, double* tr) {
  constexpr int NP = N * N;
  for (int t = threadIdx.x; t < 4 * N; t += blockDim.x) {
    const int f = t / N, k = t % N;
    const int kk = (f >= 2) ? N - 1 - k : k;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int pt = (f == 0 || f == 2) ? i * N + kk : kk * N + i;
        s += ((f == 1 || f == 2) ? MX_ER(i) : MX_EL(i)) * X[v * NP + pt];
      }
      tr[(f * MXN + k) * NV + v] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// global residual pieces

// element CTA: its q into point planes [4][NP]
template <int N>
__device__ __forceinline__ void mx_load_q(const MixDev& m, int64_t e, const double* q, const double* X, double eps,
                                          double* sQ) {
  constexpr int NP = N * N;
  const double* src = q + m.off[e];
  for (int i = threadIdx.x; i < NP * 4; i += blockDim.x) {
    double v = src[i];
    if (X) v = __dadd_rn(v, __dmul_rn(eps, X[m.off[e] + i]));
    sQ[(i % 4) * NP + i / 4] = v;
  }
}

template <int P, int KIND>
__global__ void __launch_bounds__(MXT) kmx_trace(const FrConst C, const MixDev m, const int* elems, int64_t cnt,
                                                 const double* __restrict__ q, const double* __restrict__ X,
                                                 double eps, double* __restrict__ qtr, int* bad) {
  constexpr int N = P + 1, NP = N * N;
  __shared__ double sops[MX_OPS];
  __shared__ double sQ[4 * NP];
  __shared__ double str[4 * MXN * 4];
  if (blockIdx.x >= cnt) return;
  const int64_t e = elems[blockIdx.x];
  load_ops<N>(m, sops);
  mx_load_q<N>(m, e, q, X, eps, sQ);
  __syncthreads();
  if (bad != nullptr && KT<KIND>::FLOW) {
    bool ok = true;
    for (int t = threadIdx.x; t < NP; t += blockDim.x) {
      const double x[4] = {sQ[t], sQ[NP + t], sQ[2 * NP + t], sQ[3 * NP + t]};
      ok = ok && physical(x, C.gamma);
    }
    if (!ok) atomicMin(bad, (int)e);
  }
  mx_traces<N, 4>(sops, sQ, str);
  __syncthreads();
  for (int t = threadIdx.x; t < 4 * N; t += blockDim.x) {
    const int f = t / N, k = t % N;
    const double* s = str + (f * MXN + k) * 4;
    if (bad != nullptr && KT<KIND>::FLOW && !physical(s, C.gamma)) atomicMin(bad + 1, (int)e);
    double* d = qtr + ((e * 4 + f) * MXN + k) * 4;
#pragma unroll
    for (int v = 0; v < 4; ++v) d[v] = s[v];
  }
}

// the low side's values at the high side's points: Pi (nH x nL) x
__device__ __forceinline__ void mx_up(const MixDev& m, int pH, int pL, const double* x, int nv, double* y) {
  const int nH = pH + 1, nL = pL + 1;
  if (pH == pL) {
    for (int i = 0; i < nH * nv; ++i) y[i] = x[i];
    return;
  }
  const double* Pi = xf_pi(m, pH, pL);
  for (int k = 0; k < nH; ++k)
    for (int v = 0; v < nv; ++v) {
      double s = 0.0;
      for (int l = 0; l < nL; ++l) s += Pi[k * 6 + l] * x[l * nv + v];
      y[k * nv + v] = s;
    }
}
// the high points' values restricted to the low side: Gamma (nL x nH) x
__device__ __forceinline__ void mx_down(const MixDev& m, int pH, int pL, const double* x, int nv, double* y) {
  const int nH = pH + 1, nL = pL + 1;
  if (pH == pL) {
    for (int i = 0; i < nH * nv; ++i) y[i] = x[i];
    return;
  }
  const double* Ga = xf_gamma(m, pH, pL);
  for (int l = 0; l < nL; ++l)
    for (int v = 0; v < nv; ++v) {
      double s = 0.0;
      for (int k = 0; k < nH; ++k) s += Ga[l * 6 + k] * x[k * nv + v];
      y[l * nv + v] = s;
    }
}

// one thread per face: interface flux and BR1 value (spatial.py:516-546)
template <int KIND>
__global__ void __launch_bounds__(128) kmx_face(const FrConst C, const MixDev m, const double* __restrict__ qtr,
                                                double* __restrict__ fci, double* __restrict__ wh) {
  const int64_t phi = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (phi >= m.nface) return;
  const int4 fr = m.faces[phi];
  const int fL = fr.y & 3, rev = (fr.y >> 2) & 1, bnd = (fr.y >> 3) & 1, tag = (fr.y >> 4) & 15;
  const int pL = m.deg[fr.x], nL = pL + 1;
  const double nx = m.geom[(int64_t)fr.x * 20 + 8 + 2 * fL], ny = m.geom[(int64_t)fr.x * 20 + 9 + 2 * fL];
  const Phys ph = phys_of(C);
  const double g = C.gamma;
  constexpr bool VISC = KT<KIND>::VISC;
  double a[MXN * 4], c[MXN * 4], F[MXN * 4], W[MXN * 3];
  const double* tl = qtr + ((int64_t)fr.x * 4 + fL) * MXN * 4;
  if (bnd) {  // own points, ghost state (spatial.py:508-514, 530-534, 544-546)
    for (int k = 0; k < nL; ++k) {
      double qa[4], qc[4], Fk[4];
      for (int v = 0; v < 4; ++v) qa[v] = tl[k * 4 + v];
      ghost<KIND>(qa, tag, nx, ny, C.qinf, qc);
      num_flux<KIND>(qa, qc, nx, ny, ph, Fk);
      double* d = fci + (((int64_t)fr.x * 4 + fL) * MXN + k) * 4;
      for (int v = 0; v < 4; ++v) d[v] = Fk[v];
      if (VISC) {
        double wa[3], wc[3];
        grad_vars<KIND>(qa, g, wa);
        grad_vars<KIND>(qc, g, wc);
        ghost_w<KIND>(ph, tag, wa, wc);
        double* dw = wh + (((int64_t)fr.x * 4 + fL) * MXN + k) * 3;
        for (int cc = 0; cc < 3; ++cc) dw[cc] = 0.5 * (wa[cc] + wc[cc]);
      }
    }
    return;
  }
  const int pR = m.deg[fr.z], nR = pR + 1;
  const int pH = pL > pR ? pL : pR, nH = pH + 1;
  double tr[MXN * 4];
  const double* trp = qtr + ((int64_t)fr.z * 4 + fr.w) * MXN * 4;
  for (int k = 0; k < nR; ++k)
    for (int v = 0; v < 4; ++v) tr[k * 4 + v] = trp[(rev ? nR - 1 - k : k) * 4 + v];
  double tl2[MXN * 4];
  for (int i = 0; i < nL * 4; ++i) tl2[i] = tl[i];
  mx_up(m, pH, pL, tl2, 4, a);
  mx_up(m, pH, pR, tr, 4, c);
  for (int k = 0; k < nH; ++k) num_flux<KIND>(a + 4 * k, c + 4 * k, nx, ny, ph, F + 4 * k);
  double vL[MXN * 4], vR[MXN * 4];
  mx_down(m, pH, pL, F, 4, vL);
  for (int i = 0; i < nH * 4; ++i) F[i] = -F[i];
  mx_down(m, pH, pR, F, 4, vR);
  for (int k = 0; k < nL; ++k)
    for (int v = 0; v < 4; ++v) fci[(((int64_t)fr.x * 4 + fL) * MXN + k) * 4 + v] = vL[k * 4 + v];
  for (int k = 0; k < nR; ++k)
    for (int v = 0; v < 4; ++v)
      fci[(((int64_t)fr.z * 4 + fr.w) * MXN + (rev ? nR - 1 - k : k)) * 4 + v] = vR[k * 4 + v];
  if (VISC) {
    // the viscous variables of each side's own traces, then aligned and
    // interpolated like the traces (spatial.py:541-543)
    double wl[MXN * 3], wr[MXN * 3], wa[MXN * 3], wc[MXN * 3];
    for (int k = 0; k < nL; ++k) grad_vars<KIND>(tl2 + 4 * k, g, wl + 3 * k);
    for (int k = 0; k < nR; ++k) grad_vars<KIND>(tr + 4 * k, g, wr + 3 * k);
    mx_up(m, pH, pL, wl, 3, wa);
    mx_up(m, pH, pR, wr, 3, wc);
    for (int i = 0; i < nH * 3; ++i) W[i] = 0.5 * (wa[i] + wc[i]);
    double wL[MXN * 3], wR[MXN * 3];
    mx_down(m, pH, pL, W, 3, wL);
    mx_down(m, pH, pR, W, 3, wR);
    for (int k = 0; k < nL; ++k)
      for (int cc = 0; cc < 3; ++cc) wh[(((int64_t)fr.x * 4 + fL) * MXN + k) * 3 + cc] = wL[k * 3 + cc];
    for (int k = 0; k < nR; ++k)
      for (int cc = 0; cc < 3; ++cc)
        wh[(((int64_t)fr.z * 4 + fr.w) * MXN + (rev ? nR - 1 - k : k)) * 3 + cc] = wR[k * 3 + cc];
  }
}

// element CTA: gradients (stored per point: [poff][6]) and one-sided viscous
// fluxes on own faces
template <int P, int KIND>
__global__ void __launch_bounds__(MXT) kmx_grad(const FrConst C, const MixDev m, const int* elems, int64_t cnt,
                                                const double* __restrict__ q, const double* __restrict__ X,
                                                double eps, const double* __restrict__ qtr,
                                                const double* __restrict__ wh, double* __restrict__ grad,
                                                double* __restrict__ fvn) {
  constexpr int N = P + 1, NP = N * N;
  __shared__ double sops[MX_OPS];
  __shared__ ElemGeo<N> G;
  __shared__ double sQ[4 * NP], sW[3 * NP], sWh[4 * MXN * 3], sFt[3 * NP], sGt[3 * NP], sFc[4 * MXN * 3];
  __shared__ double sgx[3 * NP], sgy[3 * NP], tgx[4 * MXN * 3], tgy[4 * MXN * 3], snrm[8];
  if (blockIdx.x >= cnt) return;
  const int64_t e = elems[blockIdx.x];
  const Phys ph = phys_of(C);
  load_ops<N>(m, sops);
  __syncthreads();
  load_geo<N>(m.geom + e * 20, sops, G);
  if (threadIdx.x < 8) snrm[threadIdx.x] = m.geom[e * 20 + 8 + threadIdx.x];
  mx_load_q<N>(m, e, q, X, eps, sQ);
  for (int i = threadIdx.x; i < 4 * MXN * 3; i += blockDim.x) sWh[i] = wh[e * 4 * MXN * 3 + i];
  __syncthreads();
  for (int t = threadIdx.x; t < NP; t += blockDim.x) {
    const double x[4] = {sQ[t], sQ[NP + t], sQ[2 * NP + t], sQ[3 * NP + t]};
    double w[3];
    grad_vars<KIND>(x, C.gamma, w);
    for (int c = 0; c < 3; ++c) sW[c * NP + t] = w[c];
  }
  __syncthreads();
  mx_gradient<N>(sops, G, sW, sWh, snrm, sFt, sGt, sFc, sgx, sgy);
  for (int t = threadIdx.x; t < NP; t += blockDim.x)
    for (int c = 0; c < 3; ++c) {
      grad[(m.poff[e] + t) * 6 + c] = sgx[c * NP + t];
      grad[(m.poff[e] + t) * 6 + 3 + c] = sgy[c * NP + t];
    }
  mx_traces<N, 3>(sops, sgx, tgx);
  mx_traces<N, 3>(sops, sgy, tgy);
  __syncthreads();
  for (int t = threadIdx.x; t < 4 * N; t += blockDim.x) {
    const int f = t / N, k = t % N;
    const double* trq = qtr + ((e * 4 + f) * MXN + k) * 4;
    double fx[4], fy[4];
    visc_flux<KIND>(trq, tgx + (f * MXN + k) * 3, tgy + (f * MXN + k) * 3, ph, fx, fy);
    double* d = fvn + ((e * 4 + f) * MXN + k) * 4;
    for (int v = 0; v < 4; ++v) d[v] = fx[v] * snrm[2 * f] + fy[v] * snrm[2 * f + 1];
  }
}

// one thread per face: the common viscous normal flux (spatial.py:559-568)
template <int KIND>
__global__ void __launch_bounds__(128) kmx_visc(const FrConst C, const MixDev m, const double* __restrict__ fvn,
                                                double* __restrict__ fcv) {
  const int64_t phi = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (phi >= m.nface) return;
  const int4 fr = m.faces[phi];
  const int fL = fr.y & 3, rev = (fr.y >> 2) & 1, bnd = (fr.y >> 3) & 1, tag = (fr.y >> 4) & 15;
  const int pL = m.deg[fr.x], nL = pL + 1;
  const double* fl = fvn + ((int64_t)fr.x * 4 + fL) * MXN * 4;
  if (bnd) {
    for (int k = 0; k < nL; ++k) {
      double* d = fcv + (((int64_t)fr.x * 4 + fL) * MXN + k) * 4;
      for (int v = 0; v < 4; ++v) d[v] = fl[k * 4 + v];
      if (KT<KIND>::FLOW && tag == T_WALL_ADIABATIC) d[3] = 0.0;
    }
    return;
  }
  const int pR = m.deg[fr.z], nR = pR + 1;
  const int pH = pL > pR ? pL : pR, nH = pH + 1;
  double x[MXN * 4], y[MXN * 4], a[MXN * 4], c[MXN * 4], val[MXN * 4];
  const double* frp = fvn + ((int64_t)fr.z * 4 + fr.w) * MXN * 4;
  for (int i = 0; i < nL * 4; ++i) x[i] = fl[i];
  for (int k = 0; k < nR; ++k)
    for (int v = 0; v < 4; ++v) y[k * 4 + v] = frp[(rev ? nR - 1 - k : k) * 4 + v];
  mx_up(m, pH, pL, x, 4, a);
  mx_up(m, pH, pR, y, 4, c);
  for (int i = 0; i < nH * 4; ++i) val[i] = 0.5 * (a[i] - c[i]);
  double vL[MXN * 4], vR[MXN * 4];
  mx_down(m, pH, pL, val, 4, vL);
  for (int i = 0; i < nH * 4; ++i) val[i] = -val[i];
  mx_down(m, pH, pR, val, 4, vR);
  for (int k = 0; k < nL; ++k)
    for (int v = 0; v < 4; ++v) fcv[(((int64_t)fr.x * 4 + fL) * MXN + k) * 4 + v] = vL[k * 4 + v];
  for (int k = 0; k < nR; ++k)
    for (int v = 0; v < 4; ++v)
      fcv[(((int64_t)fr.z * 4 + fr.w) * MXN + (rev ? nR - 1 - k : k)) * 4 + v] = vR[k * 4 + v];
}

// element CTA: volume fluxes, divergence, epilogue (spatial.py:605-629)
template <int P, int KIND>
__global__ void __launch_bounds__(MXT) kmx_asm(const FrConst C, const MixDev m, const int* elems, int64_t cnt,
                                               const double* __restrict__ q, const double* __restrict__ X,
                                               double eps, const double* __restrict__ grad,
                                               const double* __restrict__ fci, const double* __restrict__ fcv,
                                               const Epi ep, double* __restrict__ out) {
  constexpr int N = P + 1, NP = N * N;
  constexpr bool VISC = KT<KIND>::VISC;
  __shared__ double sops[MX_OPS];
  __shared__ ElemGeo<N> G;
  __shared__ double sQ[4 * NP], sFt[4 * NP], sGt[4 * NP], sFc[4 * MXN * 4];
  if (blockIdx.x >= cnt) return;
  const int64_t e = elems[blockIdx.x];
  const Phys ph = phys_of(C);
  load_ops<N>(m, sops);
  __syncthreads();
  load_geo<N>(m.geom + e * 20, sops, G);
  mx_load_q<N>(m, e, q, X, eps, sQ);
  for (int i = threadIdx.x; i < 4 * MXN * 4; i += blockDim.x)
    sFc[i] = VISC ? fci[e * 4 * MXN * 4 + i] - fcv[e * 4 * MXN * 4 + i] : fci[e * 4 * MXN * 4 + i];
  __syncthreads();
  for (int t = threadIdx.x; t < NP; t += blockDim.x) {
    const double x[4] = {sQ[t], sQ[NP + t], sQ[2 * NP + t], sQ[3 * NP + t]};
    double fx[4], fy[4];
    double r, ir, u, v, p;
    prim(x, C.gamma, r, ir, u, v, p);
    fx[0] = x[1];
    fx[1] = x[1] * u + p;
    fx[2] = x[1] * v;
    fx[3] = u * (x[3] + p);
    fy[0] = x[2];
    fy[1] = x[2] * u;
    fy[2] = x[2] * v + p;
    fy[3] = v * (x[3] + p);
    if (VISC) {
      double gx[3], gy[3], vx[4], vy[4];
      for (int c = 0; c < 3; ++c) {
        gx[c] = grad[(m.poff[e] + t) * 6 + c];
        gy[c] = grad[(m.poff[e] + t) * 6 + 3 + c];
      }
      visc_flux<KIND>(x, gx, gy, ph, vx, vy);
      for (int w = 0; w < 4; ++w) {
        fx[w] = fx[w] - vx[w];
        fy[w] = fy[w] - vy[w];
      }
    }
    for (int w = 0; w < 4; ++w) {
      sFt[w * NP + t] = G.j11[t] * fx[w] - G.j01[t] * fy[w];
      sGt[w * NP + t] = -G.j10[t] * fx[w] + G.j00[t] * fy[w];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NP; t += blockDim.x) {
    double d[4];
    mx_div_at<N, 4>(sops, G, sFt, sGt, sFc, t / N, t % N, d);
    for (int w = 0; w < 4; ++w) {
      const int64_t i = m.off[e] + t * 4 + w;
      out[i] = epi_apply(ep, i, -d[w], sQ[w * NP + t]);
    }
  }
}

// ---------------------------------------------------------------------------
// frozen records and the element-local residual

// one thread per (element, face): neighbour trace, viscous variables and
// -fvn, aligned (rev) and transferred to own points (spatial.py:700-766)
template <int KIND>
__global__ void __launch_bounds__(128) kmx_records(const FrConst C, const MixDev m, const double* __restrict__ qtr,
                                                   const double* __restrict__ fvn, double* __restrict__ rq,
                                                   double* __restrict__ rw, double* __restrict__ rf) {
  const int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (t >= m.M * 4) return;
  const int64_t e = t / 4;
  const int f = (int)(t % 4);
  const int2 lk = m.link[e * 4 + f];
  if (lk.x < 0) return;
  const int nb = lk.x, fnb = lk_face(lk.y), rev = lk_rev(lk.y);
  const int pe = m.deg[e], pn = m.deg[nb], ne = pe + 1, nn = pn + 1;
  double x[MXN * 4], w[MXN * 3], y[MXN * 4];
  const double* src = qtr + ((int64_t)nb * 4 + fnb) * MXN * 4;
  for (int k = 0; k < nn; ++k)
    for (int v = 0; v < 4; ++v) x[k * 4 + v] = src[(rev ? nn - 1 - k : k) * 4 + v];
  for (int k = 0; k < nn; ++k) grad_vars<KIND>(x + 4 * k, C.gamma, w + 3 * k);
  auto xfer = [&](const double* in, int nv, double* outp) {
    if (pn == pe) {
      for (int i = 0; i < ne * nv; ++i) outp[i] = in[i];
    } else if (pn < pe) {
      mx_up(m, pe, pn, in, nv, outp);
    } else {
      mx_down(m, pn, pe, in, nv, outp);
    }
  };
  xfer(x, 4, y);
  for (int k = 0; k < ne; ++k)
    for (int v = 0; v < 4; ++v) rq[((e * 4 + f) * MXN + k) * 4 + v] = y[k * 4 + v];
  if (KT<KIND>::VISC) {
    double wy[MXN * 3];
    xfer(w, 3, wy);
    for (int k = 0; k < ne; ++k)
      for (int c = 0; c < 3; ++c) rw[((e * 4 + f) * MXN + k) * 3 + c] = wy[k * 3 + c];
    const double* fs = fvn + ((int64_t)nb * 4 + fnb) * MXN * 4;
    for (int k = 0; k < nn; ++k)
      for (int v = 0; v < 4; ++v) x[k * 4 + v] = fs[(rev ? nn - 1 - k : k) * 4 + v];
    xfer(x, 4, y);
    for (int k = 0; k < ne; ++k)
      for (int v = 0; v < 4; ++v) rf[((e * 4 + f) * MXN + k) * 4 + v] = -y[k * 4 + v];
  }
}

// CTA per (element, state): residual of element elems[b] at state Q[b]
// with the neighbours' frozen records (spatial.py:768-853)
template <int P, int KIND>
__global__ void __launch_bounds__(MXT) kmx_local(const FrConst C, const MixDev m, const int64_t* elems, int64_t B,
                                                 const double* __restrict__ Q, const double* __restrict__ rq,
                                                 const double* __restrict__ rw, const double* __restrict__ rf,
                                                 double* __restrict__ out) {
  constexpr int N = P + 1, NP = N * N;
  constexpr bool VISC = KT<KIND>::VISC;
  __shared__ double sops[MX_OPS];
  __shared__ ElemGeo<N> G;
  __shared__ double sQ[4 * NP], str[4 * MXN * 4], sFc[4 * MXN * 4], sgh[4 * MXN * 4], snrm[8];
  __shared__ double sW[3 * NP], sWh[4 * MXN * 3], sFt[4 * NP], sGt[4 * NP], sFcs[4 * MXN * 3];
  __shared__ double sgx[3 * NP], sgy[3 * NP], tgx[4 * MXN * 3], tgy[4 * MXN * 3];
  __shared__ int2 slk[4];
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  const int64_t e = elems[b];
  const Phys ph = phys_of(C);
  load_ops<N>(m, sops);
  __syncthreads();
  load_geo<N>(m.geom + e * 20, sops, G);
  if (threadIdx.x < 8) snrm[threadIdx.x] = m.geom[e * 20 + 8 + threadIdx.x];
  if (threadIdx.x < 4) slk[threadIdx.x] = m.link[e * 4 + threadIdx.x];
  for (int i = threadIdx.x; i < NP * 4; i += blockDim.x) sQ[(i % 4) * NP + i / 4] = Q[b * NP * 4 + i];
  __syncthreads();
  mx_traces<N, 4>(sops, sQ, str);
  __syncthreads();
  // inviscid common fluxes at own points: own trace vs the frozen neighbour
  // trace or the ghost state
  for (int t = threadIdx.x; t < 4 * N; t += blockDim.x) {
    const int f = t / N, k = t % N;
    const double* qa = str + (f * MXN + k) * 4;
    double* qc = sgh + (f * MXN + k) * 4;
    if (slk[f].x < 0)
      ghost<KIND>(qa, lk_tag(slk[f].y), snrm[2 * f], snrm[2 * f + 1], C.qinf, qc);
    else
      for (int v = 0; v < 4; ++v) qc[v] = rq[((e * 4 + f) * MXN + k) * 4 + v];
    num_flux<KIND>(qa, qc, snrm[2 * f], snrm[2 * f + 1], ph, sFc + (f * MXN + k) * 4);
    if (VISC) {
      double wa[3], wc[3];
      grad_vars<KIND>(qa, C.gamma, wa);
      if (slk[f].x < 0) {
        grad_vars<KIND>(qc, C.gamma, wc);
        ghost_w<KIND>(ph, lk_tag(slk[f].y), wa, wc);
      } else {
        for (int c = 0; c < 3; ++c) wc[c] = rw[((e * 4 + f) * MXN + k) * 3 + c];
      }
      for (int c = 0; c < 3; ++c) sWh[(f * MXN + k) * 3 + c] = 0.5 * (wa[c] + wc[c]);
    }
  }
  if (VISC) {
    for (int t = threadIdx.x; t < NP; t += blockDim.x) {
      const double x[4] = {sQ[t], sQ[NP + t], sQ[2 * NP + t], sQ[3 * NP + t]};
      double w[3];
      grad_vars<KIND>(x, C.gamma, w);
      for (int c = 0; c < 3; ++c) sW[c * NP + t] = w[c];
    }
    __syncthreads();
    mx_gradient<N>(sops, G, sW, sWh, snrm, sFt, sGt, sFcs, sgx, sgy);
    mx_traces<N, 3>(sops, sgx, tgx);
    mx_traces<N, 3>(sops, sgy, tgy);
    __syncthreads();
    for (int t = threadIdx.x; t < 4 * N; t += blockDim.x) {
      const int f = t / N, k = t % N;
      double fx[4], fy[4], o[4];
      visc_flux<KIND>(str + (f * MXN + k) * 4, tgx + (f * MXN + k) * 3, tgy + (f * MXN + k) * 3, ph, fx, fy);
      for (int v = 0; v < 4; ++v) o[v] = fx[v] * snrm[2 * f] + fy[v] * snrm[2 * f + 1];
      double* fc = sFc + (f * MXN + k) * 4;
      if (slk[f].x < 0) {
        if (KT<KIND>::FLOW && lk_tag(slk[f].y) == T_WALL_ADIABATIC) o[3] = 0.0;
        for (int v = 0; v < 4; ++v) fc[v] = fc[v] - o[v];
      } else {
        for (int v = 0; v < 4; ++v) fc[v] = fc[v] - 0.5 * (o[v] + rf[((e * 4 + f) * MXN + k) * 4 + v]);
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NP; t += blockDim.x) {
    const double x[4] = {sQ[t], sQ[NP + t], sQ[2 * NP + t], sQ[3 * NP + t]};
    double fx[4], fy[4];
    double r, ir, u, v, p;
    prim(x, C.gamma, r, ir, u, v, p);
    fx[0] = x[1];
    fx[1] = x[1] * u + p;
    fx[2] = x[1] * v;
    fx[3] = u * (x[3] + p);
    fy[0] = x[2];
    fy[1] = x[2] * u;
    fy[2] = x[2] * v + p;
    fy[3] = v * (x[3] + p);
    if (VISC) {
      double gx[3], gy[3], vx[4], vy[4];
      for (int c = 0; c < 3; ++c) {
        gx[c] = sgx[c * NP + t];
        gy[c] = sgy[c * NP + t];
      }
      visc_flux<KIND>(x, gx, gy, ph, vx, vy);
      for (int w = 0; w < 4; ++w) {
        fx[w] = fx[w] - vx[w];
        fy[w] = fy[w] - vy[w];
      }
    }
    for (int w = 0; w < 4; ++w) {
      sFt[w * NP + t] = G.j11[t] * fx[w] - G.j01[t] * fy[w];
      sGt[w * NP + t] = -G.j10[t] * fx[w] + G.j00[t] * fy[w];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NP; t += blockDim.x) {
    double d[4];
    mx_div_at<N, 4>(sops, G, sFt, sGt, sFc, t / N, t % N, d);
    for (int w = 0; w < 4; ++w) out[b * NP * 4 + t * 4 + w] = -d[w];
  }
}

// ---------------------------------------------------------------------------
// host side

#define MX_GROUPS(FN, ...)                                    \
  switch (p) {                                                \
    case 0: FN<0, KIND><<<grid, MXT, 0, st>>>(__VA_ARGS__); break; \
    case 1: FN<1, KIND><<<grid, MXT, 0, st>>>(__VA_ARGS__); break; \
    case 2: FN<2, KIND><<<grid, MXT, 0, st>>>(__VA_ARGS__); break; \
    case 3: FN<3, KIND><<<grid, MXT, 0, st>>>(__VA_ARGS__); break; \
    case 4: FN<4, KIND><<<grid, MXT, 0, st>>>(__VA_ARGS__); break; \
    case 5: FN<5, KIND><<<grid, MXT, 0, st>>>(__VA_ARGS__); break; \
  }

struct MixGroups {
  const int* elems[6];  // device element lists per degree
  int64_t cnt[6];
};

__global__ void kmx_commit(int* bad, Status* st) { commit_status(bad, st); }

template <int KIND>
static int mx_residual_t(const FrConst& C, const MixDev& m, const MixGroups& gr, const double* q, const double* X,
                         double eps, const Epi& ep, double* qtr, double* fci, double* wh, double* grad, double* fvn,
                         double* fcv, double* out, int* bad, Status* stp, cudaStream_t st) {
  // out == nullptr: stop after the one-sided viscous fluxes (freeze)
  for (int p = 0; p <= 5; ++p) {
    if (!gr.cnt[p]) continue;
    const unsigned grid = (unsigned)gr.cnt[p];
    MX_GROUPS(kmx_trace, C, m, gr.elems[p], gr.cnt[p], q, X, eps, qtr, bad)
  }
  const unsigned gfac = (unsigned)((m.nface + 127) / 128);
  kmx_face<KIND><<<gfac, 128, 0, st>>>(C, m, qtr, fci, wh);
  if (KT<KIND>::VISC) {
    for (int p = 0; p <= 5; ++p) {
      if (!gr.cnt[p]) continue;
      const unsigned grid = (unsigned)gr.cnt[p];
      MX_GROUPS(kmx_grad, C, m, gr.elems[p], gr.cnt[p], q, X, eps, qtr, wh, grad, fvn)
    }
    if (out == nullptr) return (int)cudaGetLastError();
    kmx_visc<KIND><<<gfac, 128, 0, st>>>(C, m, fvn, fcv);
  }
  if (out == nullptr) return (int)cudaGetLastError();
  for (int p = 0; p <= 5; ++p) {
    if (!gr.cnt[p]) continue;
    const unsigned grid = (unsigned)gr.cnt[p];
    MX_GROUPS(kmx_asm, C, m, gr.elems[p], gr.cnt[p], q, X, eps, grad, fci, fcv, ep, out)
  }
  if (bad != nullptr) kmx_commit<<<1, 1, 0, st>>>(bad, stp);
  return (int)cudaGetLastError();
}

int mx_residual(const FrConst& C, const MixDev& m, const MixGroups& gr, const double* q, const double* X,
                double eps, const Epi& ep, double* qtr, double* fci, double* wh, double* grad, double* fvn,
                double* fcv, double* out, int* bad, Status* stp, cudaStream_t st) {
  if (m.kind == K_NS)
    return mx_residual_t<K_NS>(C, m, gr, q, X, eps, ep, qtr, fci, wh, grad, fvn, fcv, out, bad, stp, st);
  if (m.kind == K_EULER)
    return mx_residual_t<K_EULER>(C, m, gr, q, X, eps, ep, qtr, fci, wh, grad, fvn, fcv, out, bad, stp, st);
  return -3;
}

template <int KIND>
static int mx_records_t(const FrConst& C, const MixDev& m, const double* qtr, const double* fvn, double* rq,
                        double* rw, double* rf, cudaStream_t st) {
  kmx_records<KIND><<<(unsigned)((m.M * 4 + 127) / 128), 128, 0, st>>>(C, m, qtr, fvn, rq, rw, rf);
  return (int)cudaGetLastError();
}

int mx_records(const FrConst& C, const MixDev& m, const double* qtr, const double* fvn, double* rq, double* rw,
               double* rf, cudaStream_t st) {
  if (m.kind == K_NS) return mx_records_t<K_NS>(C, m, qtr, fvn, rq, rw, rf, st);
  if (m.kind == K_EULER) return mx_records_t<K_EULER>(C, m, qtr, fvn, rq, rw, rf, st);
  return -3;
}

template <int KIND>
static int mx_local_t(const FrConst& C, const MixDev& m, int p, const int64_t* elems, int64_t B, const double* Q,
                      const double* rq, const double* rw, const double* rf, double* out, cudaStream_t st) {
  const unsigned grid = (unsigned)B;
  MX_GROUPS(kmx_local, C, m, elems, B, Q, rq, rw, rf, out)
  return (int)cudaGetLastError();
}

int mx_local(const FrConst& C, const MixDev& m, int p, const int64_t* elems, int64_t B, const double* Q,
             const double* rq, const double* rw, const double* rf, double* out, cudaStream_t st) {
  if (B <= 0) return 0;
  if (m.kind == K_NS) return mx_local_t<K_NS>(C, m, p, elems, B, Q, rq, rw, rf, out, st);
  if (m.kind == K_EULER) return mx_local_t<K_EULER>(C, m, p, elems, B, Q, rq, rw, rf, out, st);
  return -3;
}

}  // namespace pmgb
