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
// Shared arrays are SoA component planes (consecutive points of a plane
// are consecutive doubles), so point-parallel accesses are conflict-free.
// BR1 reaches two elements deep, so the global residual is split at the
// two neighbour exchanges (traces, then one-sided viscous fluxes).
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "pmgb_internal.cuh"
#include "fr_device.cuh"

#ifndef PMGB_FVN_REGS_P2
#define PMGB_FVN_REGS_P2 64
#endif
#ifndef PMGB_FVN_REGS_P3   // p = 3: 72 (R 118 -> 111 us at config 4, profiles/r1/ab_fvn_regs_r1q.log)
#define PMGB_FVN_REGS_P3 72
#endif
#ifndef PMGB_FVN_REGS
#define PMGB_FVN_REGS 64
#endif
#ifndef PMGB_FVN_REGS_P5
#define PMGB_FVN_REGS_P5 80
#endif
#ifndef PMGB_IDET_SMEM
#define PMGB_IDET_SMEM 0   // 1/det J once per point in shared memory (measured: slower)
#endif
#ifndef PMGB_TRACE_REGS
#define PMGB_TRACE_REGS 40
#endif

namespace pmgb {

// ---------------------------------------------------------------------------
// shared-memory layout (in doubles) per CTA.  Planes: point planes hold
// NPT = E*NP values (index el*NP + pt), face planes NFT = E*4N values
// (index el*4N + f*N + k).

template <int P, int KIND>
struct SL {
  using B = BC<P>;
  using T = KT<KIND>;
  static constexpr int E = B::EPB, N = B::N, NP = B::NP, NV = T::NV, NW = T::NW;
  static constexpr int NPT = E * NP, NFT = E * 4 * N;
  static constexpr int OP = 0;                    // D(36) eL eR lL lR xg (6 each)
  static constexpr int G = 72;                    // [E][20] geometry records
  static constexpr int Q = G + E * 20;            // [NV] point planes
  static constexpr int W = Q + NV * NPT;          // [NW] point planes   viscous variables
  static constexpr int WH = W + NW * NPT;         // [NW] face planes    BR1 common value (CCW k)
  static constexpr int CG = WH + NW * NFT;        // [2NW] face planes   gradient lifting (line j)
  static constexpr int FC = CG + 2 * NW * NFT;    // [NV] face planes    common flux (CCW k)
  static constexpr int FT = FC + NV * NFT;        // [NV] point planes   contravariant flux xi
  static constexpr int GT = FT + NV * NPT;        // [NV] point planes   contravariant flux eta
  static constexpr int CF = CG;                   // [NV] face planes    flux lifting (aliases CG: dead by then)
  static constexpr int END_ASM = GT + NV * NPT;
  static constexpr int GR = END_ASM;              // [2NW] point planes  gradients (local pipeline)
  static constexpr int TR = GR + 2 * NW * NPT;    // [NV] face planes    own traces (local pipeline)
  static constexpr int R0 = TR + NV * NFT;        // [NP*NV]             unperturbed local residual
  static constexpr int END_LOCAL = R0 + NP * NV;
  static constexpr int OVQ = END_LOCAL;           // [E][N][NV]  face-record override: neighbour trace
  static constexpr int OVF = OVQ + E * N * NV;    // [E][N][NV]  face-record override: neighbour fvn
  static constexpr size_t BYTES_COUPLING = sizeof(double) * (OVF + E * N * NV);
  // Padded point planes of k_fvn / k_assemble_async (bank spread): point
  // (el, a, b) of a plane at el*ES + a*RS + b, planes PS apart.  The strides
  // minimise modelled shared wavefronts over the point-, row- and
  // column-thread patterns of both kernels (even N needs them most).
  static constexpr int RS = N;
  static constexpr int ES_T = P == 3 ? 17 : N * RS;
  static constexpr int ES = ES_T > N * RS ? ES_T : N * RS;
  // p=4 and p=5 measured fastest unpadded (the model's gains there are
  // smaller than the extra index arithmetic and spills they cost)
  static constexpr int PS_T = P == 1 ? 129 : P == 2 ? 132 : P == 3 ? 139 : 0;
  static constexpr int PS = PS_T > E * ES ? PS_T : E * ES;
  __host__ __device__ static constexpr int pix(int el, int a, int b) { return el * ES + a * RS + b; }
  static constexpr bool PADDED = !(RS == N && ES == NP);
  __host__ __device__ static constexpr int pix(int t) { return PADDED ? pix(t / NP, (t % NP) / N, t % N) : t; }
  // k_fvn: padded point planes Q, W; face planes padded to an element
  // stride of 4N+1; the gradient planes 16-byte aligned for the block copy
  static constexpr int NFS = 4 * N + 1, NFTP = E * NFS;
  static constexpr int F_Q = G + E * 20;          // [NV] padded point planes
  static constexpr int F_W = F_Q + NV * PS;       // [NW] padded point planes   viscous variables
  static constexpr int F_WH = F_W + NW * PS;      // [NW] padded face planes  BR1 common value
  static constexpr int F_GF = F_WH + NW * NFTP;   // [2NW] padded face planes gradient traces
  static constexpr int GR_FVN = (F_GF + 2 * NW * NFTP + 1) & ~1;  // [2NW] padded point planes
  // k_assemble_async: AoS q (cp.async), face fluxes, padded flux planes
  static constexpr int P_FT = Q + NV * NPT + NV * NFT;  // after A_FC (AoS q, face fluxes)
  static constexpr int P_GT = P_FT + NV * PS;
  static constexpr int P_ID = P_GT + NV * PS;     // [1] padded point plane  1/det J
  static constexpr size_t BYTES_ASYNC = sizeof(double) * (P_ID + (PMGB_IDET_SMEM ? PS : 0));
  // compact layout of k_assemble (gradients come from k_fvn)
  static constexpr int A_FC = Q + NV * NPT;
  static constexpr int A_FT = A_FC + NV * NFT;
  static constexpr int A_GT = A_FT + NV * NPT;
  static constexpr int A_CF = A_GT + NV * NPT;
  static constexpr size_t BYTES_TRACE = sizeof(double) * (Q + NV * NPT);
  static constexpr size_t BYTES_FVN = sizeof(double) * (GR_FVN + 2 * NW * PS);
  static constexpr size_t BYTES_ASM = sizeof(double) * (A_CF + NV * NFT);
  static constexpr size_t BYTES_LOCAL = sizeof(double) * END_LOCAL;
  static_assert(2 * NW >= NV || true, "CF alias");
};

template <int P> struct MinBlocks {
  static constexpr int cap(int v) { return v < 1 ? 1 : (v > 32 ? 32 : v); }
  static constexpr int ASM = cap(65536 / (BC<P>::THREADS * PMGB_REG_TARGET));
  static constexpr int ASM_R = cap(65536 / (BC<P>::THREADS * (P == 5   ? PMGB_REG_TARGET_R_P5
                                                             : P == 3 ? PMGB_REG_TARGET_R_P3
                                                                      : PMGB_REG_TARGET_R)));
  static constexpr int ASM_K = cap(65536 / (BC<P>::THREADS * (P == 5   ? PMGB_REG_TARGET_K_P5
                                                             : P == 3 ? PMGB_REG_TARGET_K_P3
                                                                      : PMGB_REG_TARGET_K)));
  static constexpr int FVN = cap(65536 / (BC<P>::THREADS * (P == 5   ? PMGB_FVN_REGS_P5
                                                           : P == 3 ? PMGB_FVN_REGS_P3
                                                           : P == 2 ? PMGB_FVN_REGS_P2
                                                                    : PMGB_FVN_REGS)));
  static constexpr int TRACE = cap(65536 / (BC<P>::THREADS * PMGB_TRACE_REGS));
  static constexpr int BLK = cap(65536 / (BC<P>::THREADS * PMGB_BLOCKS_REGS));
};

struct Ops {
  const double* D;
  const double* eL;
  const double* eR;
  const double* lL;
  const double* lR;
  const double* xg;
};

template <int TH>
__device__ __forceinline__ Ops stage_ops(const FrConst& C, double* sm) {
  for (int i = threadIdx.x; i < 66; i += TH) {
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

// ---------------------------------------------------------------------------
// staging helpers

// element-major AoS global (E elements from e0) -> SoA point planes.
// NV = 4: one thread per point, two 16-byte loads (rows are 32 B aligned).
template <int P, int NV>
__device__ __forceinline__ void load_points(const double* __restrict__ src, int64_t e0, int64_t M, double* sQ) {
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB, NPT = E * NP;
  if constexpr (NV == 4) {
    const int64_t lim = (M - e0) * NP;
    const double2* base = reinterpret_cast<const double2*>(src + e0 * NP * 4);
    for (int g = threadIdx.x; g < NPT; g += BC<P>::THREADS) {
      double2 a = make_double2(1.0, 1.0), b = make_double2(1.0, 1.0);
      if (g < lim) {
        a = __ldg(base + 2 * g);
        b = __ldg(base + 2 * g + 1);
      }
      sQ[g] = a.x;
      sQ[NPT + g] = a.y;
      sQ[2 * NPT + g] = b.x;
      sQ[3 * NPT + g] = b.y;
    }
  } else {
    const int64_t lim = (M - e0) * NP * NV;
    const double* base = src + e0 * NP * NV;
    for (int i = threadIdx.x; i < NPT * NV; i += BC<P>::THREADS) {
      const int v = i % NV, g = i / NV;
      sQ[v * NPT + g] = (i < lim) ? __ldg(base + i) : 1.0;
    }
  }
}

// element-major AoS global -> padded SoA point planes (SL::pix layout)
template <int P, int NV, class L>
__device__ __forceinline__ void load_points_pad(const double* __restrict__ src, int64_t e0, int64_t M, double* sQ) {
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB, NPT = E * NP;
  if constexpr (NV == 4) {
    const int64_t lim = (M - e0) * NP;
    const double2* base = reinterpret_cast<const double2*>(src + e0 * NP * 4);
    for (int g = threadIdx.x; g < NPT; g += BC<P>::THREADS) {
      double2 a = make_double2(1.0, 1.0), b = make_double2(1.0, 1.0);
      if (g < lim) {
        a = __ldg(base + 2 * g);
        b = __ldg(base + 2 * g + 1);
      }
      const int d = L::pix(g);
      sQ[d] = a.x;
      sQ[L::PS + d] = a.y;
      sQ[2 * L::PS + d] = b.x;
      sQ[3 * L::PS + d] = b.y;
    }
  } else {
    const int64_t lim = (M - e0) * NP * NV;
    const double* base = src + e0 * NP * NV;
    for (int i = threadIdx.x; i < NPT * NV; i += BC<P>::THREADS) {
      const int v = i % NV, g = i / NV;
      sQ[v * L::PS + L::pix(g)] = (i < lim) ? __ldg(base + i) : 1.0;
    }
  }
}

template <int P>
__device__ __forceinline__ void load_links(const int2* __restrict__ link, int64_t e0, int64_t M, int2* sLK) {
  constexpr int E = BC<P>::EPB;
  const int64_t lim = (M - e0) * 4;
  for (int i = threadIdx.x; i < E * 4; i += BC<P>::THREADS) sLK[i] = (i < lim) ? link[e0 * 4 + i] : make_int2(-1, 0);
}

template <int P>
__device__ __forceinline__ void load_geom(const double* __restrict__ geom, int64_t e0, int64_t M, double* sG) {
  constexpr int E = BC<P>::EPB;
  const int64_t lim = (M - e0) * 20;
  const double* base = geom + e0 * 20;
  for (int i = threadIdx.x; i < E * 20; i += BC<P>::THREADS) sG[i] = (i < lim) ? __ldg(base + i) : 0.0;
}

// Interpolation line of face f, point k: points base + i * stride, i < N
struct Line {
  int base, stride;
  const double* w;
};
template <int N>
__device__ __forceinline__ Line face_line(const Ops& op, int f, int k) {
  Line L;
  L.base = f == 0 ? k : f == 1 ? k * N : f == 2 ? (N - 1 - k) : (N - 1 - k) * N;
  L.stride = (f == 0 || f == 2) ? N : 1;
  L.w = (f == 0 || f == 3) ? op.eL : op.eR;
  return L;
}

template <int N>
__device__ __forceinline__ double line_sum(const Line& L, const double* plane_el) {
  double s = 0.0;
  const double* x = plane_el + L.base;
#pragma unroll
  for (int i = 0; i < N; ++i) s += L.w[i] * x[i * L.stride];
  return s;
}

// trace of one point plane (already offset to the element) at face (f, k)
template <int N>
__device__ __forceinline__ double line_sum(const Ops& op, const double* plane_el, int f, int k) {
  return line_sum<N>(face_line<N>(op, f, k), plane_el);
}

template <int NV>
__device__ __forceinline__ void ld_face(const double* __restrict__ src, double* out) {
  if constexpr (NV == 4) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(src));
    const double2 b = __ldg(reinterpret_cast<const double2*>(src) + 1);
    out[0] = a.x;
    out[1] = a.y;
    out[2] = b.x;
    out[3] = b.y;
  } else {
    out[0] = __ldg(src);
  }
}

template <int NV>
__device__ __forceinline__ void st_face(double* dst, const double* v) {
  if constexpr (NV == 4) {
    reinterpret_cast<double2*>(dst)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2*>(dst)[1] = make_double2(v[2], v[3]);
  } else {
    dst[0] = v[0];
  }
}

// ---------------------------------------------------------------------------
// BR1 gradient pieces (spatial.py:594-603 via _divergence 407-430)

// face thread: lifting terms of the x and y gradients at (f, k) -> line j
template <int P, int KIND>
__device__ __forceinline__ void grad_corrections(const Ops& op, const double* sW, const double* sG_el,
                                                 const double* sWH, double* sCG, int el, int f, int k) {
  constexpr int N = P + 1, NW = KT<KIND>::NW;
  constexpr int NPT = SL<P, KIND>::NPT, NFT = SL<P, KIND>::NFT, NP = N * N;
  const Metric mt = metric(sG_el);
  const double nx = sG_el[8 + 2 * f], ny = sG_el[9 + 2 * f], js = sG_el[16 + f];
  const double sgn = (f == 1 || f == 2) ? 1.0 : -1.0;
  const int j = (f >= 2) ? N - 1 - k : k;
  const bool xiline = (f == 1 || f == 3);
  const double* w = (f == 0 || f == 3) ? op.eL : op.eR;
  double lx[NW], ly[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c) lx[c] = ly[c] = 0.0;
  const Line L = face_line<N>(op, f, k);
  if (mt.affine()) {
    const double fxx = xiline ? mt.d0 : -mt.b0;
    const double fyy = xiline ? -mt.c0 : mt.a0;
#pragma unroll
    for (int c = 0; c < NW; ++c) {
      const double t = line_sum<N>(L, sW + c * NPT + el * NP);
      lx[c] = fxx * t;
      ly[c] = fyy * t;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double x = op.xg[i];
      // x-gradient: Ft = J11 W (xi lines), Gt = -J10 W (eta lines)
      // y-gradient: Ft = -J01 W,           Gt =  J00 W
      const double fxx = xiline ? mt.J11(x) : -mt.J10(x);
      const double fyy = xiline ? -mt.J01(x) : mt.J00(x);
      const int p = el * NP + L.base + i * L.stride;
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        const double Wv = sW[c * NPT + p];
        lx[c] += w[i] * (fxx * Wv);
        ly[c] += w[i] * (fyy * Wv);
      }
    }
  }
  const int fi = el * 4 * N + f * N + k;
  const int fj = el * 4 * N + f * N + j;
#pragma unroll
  for (int c = 0; c < NW; ++c) {
    const double wh = sWH[c * NFT + fi];
    sCG[c * NFT + fj] = sgn * js * (nx * wh) - lx[c];
    sCG[(NW + c) * NFT + fj] = sgn * js * (ny * wh) - ly[c];
  }
}

// point thread: corrected gradients at (a, b)
template <int P, int KIND>
__device__ __forceinline__ void gradient_at(const Ops& op, const double* sW, const double* sG_el,
                                            const double* sCG, int el, int a, int b, double* gx, double* gy) {
  constexpr int N = P + 1, NW = KT<KIND>::NW;
  constexpr int NPT = SL<P, KIND>::NPT, NFT = SL<P, KIND>::NFT, NP = N * N;
  const Metric mt = metric(sG_el);
  double sx[NW], sy[NW], dx[NW], dy[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c) sx[c] = sy[c] = dx[c] = dy[c] = 0.0;
  const int base = el * NP;
  if (mt.affine()) {
    // parallelogram element: J constant, factor it out of the line sums
    double Sr[NW], Sc[NW];
#pragma unroll
    for (int c = 0; c < NW; ++c) Sr[c] = Sc[c] = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double Db = op.D[b * N + i], Da = op.D[a * N + i];
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        Sr[c] += Db * sW[c * NPT + base + a * N + i];
        Sc[c] += Da * sW[c * NPT + base + i * N + b];
      }
    }
#pragma unroll
    for (int c = 0; c < NW; ++c) {
      sx[c] = mt.d0 * Sr[c];
      sy[c] = -mt.c0 * Sr[c];
      dx[c] = -mt.b0 * Sc[c];
      dy[c] = mt.a0 * Sc[c];
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double Db = op.D[b * N + i], Da = op.D[a * N + i];
      const double xi = op.xg[i];
      const double j11 = mt.J11(xi), j01 = mt.J01(xi);  // row line: xi_i
      const double j10 = mt.J10(xi), j00 = mt.J00(xi);  // column line: eta_i
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        const double Wr = sW[c * NPT + base + a * N + i];
        const double Wc = sW[c * NPT + base + i * N + b];
        sx[c] += Db * (j11 * Wr);
        sy[c] += Db * (-j01 * Wr);
        dx[c] += Da * (-j10 * Wc);
        dy[c] += Da * (j00 * Wc);
      }
    }
  }
  const double xa = op.xg[a], xb = op.xg[b];
  const double idet = rcp(mt.J00(xa) * mt.J11(xb) - mt.J01(xb) * mt.J10(xa));
  const int f0 = el * 4 * N;
  const double lRb = op.lR[b], lLb = op.lL[b], lRa = op.lR[a], lLa = op.lL[a];
#pragma unroll
  for (int c = 0; c < NW; ++c) {
    const double* cx = sCG + c * NFT + f0;
    const double* cy = sCG + (NW + c) * NFT + f0;
    double vx = sx[c] + dx[c];
    vx = vx + lRb * cx[1 * N + a];
    vx = vx - lLb * cx[3 * N + a];
    vx = vx + lRa * cx[2 * N + b];
    vx = vx - lLa * cx[0 * N + b];
    double vy = sy[c] + dy[c];
    vy = vy + lRb * cy[1 * N + a];
    vy = vy - lLb * cy[3 * N + a];
    vy = vy + lRa * cy[2 * N + b];
    vy = vy - lLa * cy[0 * N + b];
    gx[c] = vx * idet;
    gy[c] = vy * idet;
  }
}

// point thread: total flux (inviscid - viscous), transformed
template <int P, int KIND>
__device__ __forceinline__ void point_fluxes(const double* q, const double* gx, const double* gy,
                                             const Phys& ph, const Metric& mt, double xa, double xb,
                                             double* Ft, double* Gt) {
  constexpr int NV = KT<KIND>::NV;
  double fx[NV], fy[NV];
  if constexpr (KT<KIND>::FLOW) {
    double r, ir, u, v, p;
    prim(q, ph.gamma, r, ir, u, v, p);
    fx[0] = q[1];
    fx[1] = q[1] * u + p;
    fx[2] = q[1] * v;
    fx[3] = u * (q[3] + p);
    fy[0] = q[2];
    fy[1] = q[2] * u;
    fy[2] = q[2] * v + p;
    fy[3] = v * (q[3] + p);
    if constexpr (KT<KIND>::VISC) {
      const double d = gx[0] + gy[1];
      const double txx = ph.mu * (2.0 * gx[0] - (2.0 / 3.0) * d);
      const double tyy = ph.mu * (2.0 * gy[1] - (2.0 / 3.0) * d);
      const double txy = ph.mu * (gy[0] + gx[1]);
      fx[1] = fx[1] - txx;
      fx[2] = fx[2] - txy;
      fx[3] = fx[3] - (u * txx + v * txy + ph.kappa * gx[2]);
      fy[1] = fy[1] - txy;
      fy[2] = fy[2] - tyy;
      fy[3] = fy[3] - (u * txy + v * tyy + ph.kappa * gy[2]);
      fx[0] = fx[0] - 0.0;
      fy[0] = fy[0] - 0.0;
    }
  } else {
    fx[0] = ph.ax * q[0];
    fy[0] = ph.ay * q[0];
    if constexpr (KT<KIND>::VISC) {
      fx[0] = fx[0] - ph.diff * gx[0];
      fy[0] = fy[0] - ph.diff * gy[0];
    }
  }
  const double j00 = mt.J00(xa), j10 = mt.J10(xa), j01 = mt.J01(xb), j11 = mt.J11(xb);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    Ft[v] = j11 * fx[v] - j01 * fy[v];
    Gt[v] = -j10 * fx[v] + j00 * fy[v];
  }
}

// face thread: FR lifting term of the flux divergence, line j
template <int P, int KIND>
__device__ __forceinline__ void flux_corrections(const Ops& op, const double* sFT, const double* sGT,
                                                 const double* sG_el, const double* Fc, double* sCF,
                                                 int el, int f, int k) {
  constexpr int N = P + 1, NV = KT<KIND>::NV, NP = N * N;
  constexpr int NPT = SL<P, KIND>::NPT, NFT = SL<P, KIND>::NFT;
  const double js = sG_el[16 + f];
  const double sgn = (f == 1 || f == 2) ? 1.0 : -1.0;
  const int j = (f >= 2) ? N - 1 - k : k;
  const double* X = (f == 1 || f == 3) ? sFT : sGT;
  const int fj = el * 4 * N + f * N + j;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double l = line_sum<N>(op, X + v * NPT + el * NP, f, k);
    sCF[v * NFT + fj] = sgn * js * Fc[v] - l;
  }
}

// point thread: -div / det (spatial.py:407-430, 627)
template <int P, int KIND>
__device__ __forceinline__ void divergence_at(const Ops& op, const double* sFT, const double* sGT,
                                              const double* sCF, const Metric& mt, int el, int a, int b,
                                              double* R) {
  constexpr int N = P + 1, NV = KT<KIND>::NV, NP = N * N;
  constexpr int NPT = SL<P, KIND>::NPT, NFT = SL<P, KIND>::NFT;
  double s[NV], t[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) s[v] = t[v] = 0.0;
  const int base = el * NP;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double Db = op.D[b * N + i], Da = op.D[a * N + i];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      s[v] += Db * sFT[v * NPT + base + a * N + i];
      t[v] += Da * sGT[v * NPT + base + i * N + b];
    }
  }
  const double xa = op.xg[a], xb = op.xg[b];
  const double idet = rcp(mt.J00(xa) * mt.J11(xb) - mt.J01(xb) * mt.J10(xa));
  const int f0 = el * 4 * N;
  const double lRb = op.lR[b], lLb = op.lL[b], lRa = op.lR[a], lLa = op.lL[a];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double* cf = sCF + v * NFT + f0;
    double d = s[v] + t[v];
    d = d + lRb * cf[1 * N + a];
    d = d - lLb * cf[3 * N + a];
    d = d + lRa * cf[2 * N + b];
    d = d - lLa * cf[0 * N + b];
    R[v] = -(d * idet);
  }
}

template <int NV, int NPT>
__device__ __forceinline__ void gather_point(const double* sQ, int t, double* q) {
#pragma unroll
  for (int v = 0; v < NV; ++v) q[v] = sQ[v * NPT + t];
}

// ---------------------------------------------------------------------------
// phase 1: traces (+ optional q + eps X prologue, + physicality flags)

template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS, MinBlocks<P>::TRACE)
k_trace(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ X,
        double eps, double* __restrict__ qp, double* __restrict__ qtr, int* __restrict__ bad) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB, NV = KT<KIND>::NV;
  constexpr int NPT = L::NPT;
  const Ops op = stage_ops<BC<P>::THREADS>(C, sm);
  double* sQ = sm + L::Q;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int64_t M = m.M;
  if (X == nullptr) {
    load_points<P, NV>(q, e0, M, sQ);
  } else {
    // q + eps * X, rounded as the reference does (newton_krylov.py:76)
    const int64_t lim = (M - e0) * NP * NV;
    const double* qb = q + e0 * NP * NV;
    const double* xb = X + e0 * NP * NV;
    double* pb = qp + e0 * NP * NV;
    for (int i = threadIdx.x; i < NPT * NV; i += BC<P>::THREADS) {
      double v = 1.0;
      if (i < lim) {
        v = __dadd_rn(__ldg(qb + i), __dmul_rn(eps, __ldg(xb + i)));
        pb[i] = v;
      }
      sQ[(i % NV) * NPT + i / NV] = v;
    }
  }
  __syncthreads();
  const double g = C.gamma;
  if constexpr (KT<KIND>::FLOW) {
    if (bad != nullptr) {
      const int t = threadIdx.x;
      if (t < NPT) {
        const int64_t e = e0 + t / NP;
        double qq[NV];
        gather_point<NV, NPT>(sQ, t, qq);
        if (e < M && !physical(qq, g)) atomicMin(bad, (int)e);
      }
    }
  }
  for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = e0 + el;
    if (e >= M) continue;
    double tr[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = line_sum<N>(op, sQ + v * NPT + el * NP, f, k);
    if constexpr (KT<KIND>::FLOW) {
      if (bad != nullptr && !physical(tr, g)) atomicMin(bad + 1, (int)e);
    }
    st_face<NV>(qtr + ((e * 4 + f) * N + k) * NV, tr);
  }
}

// Phase 1 by line threads (4 conserved variables): thread (element, line,
// direction) reads one row (contiguous N x 4 doubles) or column of q --
// forming q + eps X on the fly with the reference's rounding -- and writes
// the two face traces at that line's ends.  Row threads also check the
// points of their row and write the perturbed state.  No shared memory,
// no barrier.
// HASX: the Jv forms (q + eps X, written to qp) are their own instantiation:
// the plain trace fits 64 registers (8 CTAs/SM), the Jv one runs best
// without a register cap (R 164.0 -> 162.1 us, Jv 206.7 -> 198.9 us at
// config 2, profiles/r1/ab_trace_regs_r1m.log)
template <int P, int KIND, bool HASX = false>
__global__ void __launch_bounds__(128, HASX ? 1 : 8)
k_trace_lines(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ X,
              double eps, double* __restrict__ qp, double* __restrict__ qtr, int* __restrict__ bad) {
  constexpr int N = P + 1, NP = N * N, NV = 4;
  pdl_trigger();
  const int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (t >= m.M * 2 * N) return;
  const int64_t e = t / (2 * N);
  const int r = (int)(t - e * 2 * N);
  const bool row = r < N;
  const int line = row ? r : r - N;
  const int stride = row ? NV : N * NV;  // between consecutive points of the line
  const int64_t base = e * NP * NV + (row ? (int64_t)line * N * NV : (int64_t)line * NV);
  double v[N][NV];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(q + base + i * stride));
    const double2 b = __ldg(reinterpret_cast<const double2*>(q + base + i * stride) + 1);
    v[i][0] = a.x;
    v[i][1] = a.y;
    v[i][2] = b.x;
    v[i][3] = b.y;
  }
  if (HASX) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double2 a = __ldg(reinterpret_cast<const double2*>(X + base + i * stride));
      const double2 b = __ldg(reinterpret_cast<const double2*>(X + base + i * stride) + 1);
      v[i][0] = __dadd_rn(v[i][0], __dmul_rn(eps, a.x));
      v[i][1] = __dadd_rn(v[i][1], __dmul_rn(eps, a.y));
      v[i][2] = __dadd_rn(v[i][2], __dmul_rn(eps, b.x));
      v[i][3] = __dadd_rn(v[i][3], __dmul_rn(eps, b.y));
    }
    if (row) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double2* o = reinterpret_cast<double2*>(qp + base + i * stride);
        o[0] = make_double2(v[i][0], v[i][1]);
        o[1] = make_double2(v[i][2], v[i][3]);
      }
    }
  }
  const double g = C.gamma;
  if (bad != nullptr && row) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) ok = ok && physical(v[i], g);
    if (!ok) atomicMin(bad, (int)e);
  }
  // rows: face 1 (xi=+1) point k=line, face 3 (xi=-1) point k=N-1-line
  // cols: face 2 (eta=+1) point k=N-1-line, face 0 (eta=-1) point k=line
  double tp[NV], tm[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    double sp = 0.0, sm = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      sp += C.eR[i] * v[i][c];
      sm += C.eL[i] * v[i][c];
    }
    tp[c] = sp;
    tm[c] = sm;
  }
  const int fp = row ? 1 : 2, fm = row ? 3 : 0;
  const int kp = row ? line : N - 1 - line, km = row ? N - 1 - line : line;
  if (bad != nullptr && !(physical(tp, g) && physical(tm, g))) atomicMin(bad + 1, (int)e);
  st_face<NV>(qtr + ((e * 4 + fp) * N + kp) * NV, tp);
  st_face<NV>(qtr + ((e * 4 + fm) * N + km) * NV, tm);
}

// ---------------------------------------------------------------------------
// phase 2: one-sided viscous normal flux on every face (spatial.py:536-557)

template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS, MinBlocks<P>::FVN)
k_fvn(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
      double* __restrict__ fvn, double* __restrict__ grad, int q_dep) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW, NPT = L::NPT, NFS = L::NFS, NFTP = L::NFTP;
  constexpr int PS = L::PS, ES = L::ES, RS = L::RS;
  pdl_trigger();
  const Ops op = stage_ops<BC<P>::THREADS>(C, sm);
  double* sQ = sm + L::F_Q;
  double* sG = sm + L::G;
  double* sW = sm + L::F_W;
  double* sWH = sm + L::F_WH;
  double* sGR = sm + L::GR_FVN;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int64_t M = m.M;
  const Phys ph = phys_of(C);
  // Prologue: q / geometry into shared memory and the face-trace gathers
  // (own + neighbour) into registers, all before the first barrier.
  constexpr bool ONE_FACE = (E * NF <= BC<P>::THREADS);
  const int t0 = threadIdx.x;
  // q_dep: q is the q + eps X written by the preceding k_trace_lines (Jv
  // forms), so it may only be read after the dependency wait
  if (!q_dep) load_points_pad<P, NV, L>(q, e0, M, sQ);
  load_geom<P>(m.geom, e0, M, sG);
  double tr[NV], nb[NV];
  int2 lk = make_int2(-1, 0);
  bool face_live = false;
  int fel = 0, ff = 0;
  // the link table is static mesh data: fetch it before the dependency wait
  if constexpr (ONE_FACE) {
    if (t0 < E * NF) {
      fel = t0 / NF;
      ff = (t0 % NF) / N;
      face_live = e0 + fel < M;
      if (face_live) lk = m.link[(e0 + fel) * 4 + ff];
    }
  }
  pdl_wait();  // traces (and for Jv the perturbed state) come from k_trace
  if (q_dep) load_points_pad<P, NV, L>(q, e0, M, sQ);
  if constexpr (ONE_FACE) {
    if (t0 < E * NF) {
      const int fk = (t0 % NF) % N;
      const int64_t e = e0 + fel;
      if (face_live) {
        const bool interior = lk.x >= 0;
        const int kk = lk_rev(lk.y) ? N - 1 - fk : fk;
        const int64_t own = ((e * 4 + ff) * N + fk) * NV;
        const int64_t nbi = interior ? (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV : own;
        ld_face<NV>(qtr + own, tr);
        ld_face<NV>(qtr + nbi, nb);
      }
    }
  }
  __syncthreads();
  // point stage: viscous variables, and 1/det J once per point into the
  // (now dead) q plane 0 for the column pass
  double* sID = sQ;
  if (t0 < NPT) {
    double qq[NV], w[NW];
    const int px0 = L::pix(t0);
#pragma unroll
    for (int v = 0; v < NV; ++v) qq[v] = sQ[v * PS + px0];
    grad_vars<KIND>(qq, ph.gamma, w);
#pragma unroll
    for (int c = 0; c < NW; ++c) sW[c * PS + px0] = w[c];
    if constexpr (PMGB_IDET_SMEM) {
      const int el = t0 / NP, pt = t0 % NP;
      const Metric mt = metric(sG + el * 20);
      const double xa = C.xg[pt / N], xb = C.xg[pt % N];
      sID[px0] = rcp(mt.J00(xa) * mt.J11(xb) - mt.J01(xb) * mt.J10(xa));
    }
  }
  auto face_avg = [&](int t, int el, int f, int2 lkk, double* tr_, double* nb_) {
    if (lkk.x < 0) {
      const double* gq = sG + el * 20;
      ghost<KIND>(tr_, lk_tag(lkk.y), gq[8 + 2 * f], gq[9 + 2 * f], C.qinf, nb_);
    }
    double wa[NW], wc[NW];
    grad_vars<KIND>(tr_, ph.gamma, wa);
    grad_vars<KIND>(nb_, ph.gamma, wc);
    if (lkk.x < 0) ghost_w<KIND>(ph, lk_tag(lkk.y), wa, wc);
    const bool inter = lkk.x >= 0, lft = inter && lk_left(lkk.y);
#pragma unroll
    for (int c = 0; c < NW; ++c) sWH[c * NFTP + el * NFS + (t - el * NF)] = common_w(ph, inter, lft, wa[c], wc[c]);
  };
  if constexpr (ONE_FACE) {
    if (face_live) face_avg(t0, fel, ff, lk, tr, nb);
  } else {
    for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
      const int el = t / NF, r = t % NF, f = r / N, k = r % N;
      const int64_t e = e0 + el;
      if (e >= M) continue;
      const int2 lkk = m.link[e * 4 + f];
      const bool interior = lkk.x >= 0;
      const int kk = lk_rev(lkk.y) ? N - 1 - k : k;
      const int64_t own = ((e * 4 + f) * N + k) * NV;
      const int64_t nbi = interior ? (((int64_t)lkk.x * 4 + lk_face(lkk.y)) * N + kk) * NV : own;
      double tr2[NV], nb2[NV];
      ld_face<NV>(qtr + own, tr2);
      ld_face<NV>(qtr + nbi, nb2);
      face_avg(t, el, f, lkk, tr2, nb2);
    }
  }
  __syncthreads();
  // BR1 gradients by line threads (element, line, viscous variable):
  //  rows : x-part   sum_i D[b][i] J11(xi_i) W[a][i] + lR[b] cx1 - lL[b] cx3 (and y with -J01)
  //  cols : eta-part sum_i D[a][i] (-J10 | J00)(eta_i) W[i][b] + lR[a] c2 - lL[a] c0, then / det
  // c_f = +-js_f n_f What_f - (trace of the metric-weighted W on face f)  (spatial.py:594-603)
  constexpr int TH = BC<P>::THREADS;
  constexpr int NLG = E * N * NW;
  double* sPX = sGR;            // [NW][PS] x partials, then gx
  double* sPY = sGR + NW * PS;  // [NW][PS] y partials, then gy
  // pass 1, rows: thread t = (c, el, a) with a fastest, so the row it reads
  // and writes starts at N * t (stride N odd: no bank conflicts)
  for (int t = t0; t < NLG; t += TH) {
    const int c = t / (E * N), el = (t / N) % E, a = t % N;
    const double* gq = sG + el * 20;
    const Metric mt = metric(gq);
    const double* Wr = sW + c * PS + el * ES + a * RS;
    double wx[N], wy[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double x = Wr[i], xi = C.xg[i];
      wx[i] = mt.J11(xi) * x;
      wy[i] = -mt.J01(xi) * x;
    }
    double tx1 = 0.0, ty1 = 0.0, tx3 = 0.0, ty3 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      tx1 += C.eR[i] * wx[i];
      ty1 += C.eR[i] * wy[i];
      tx3 += C.eL[i] * wx[i];
      ty3 += C.eL[i] * wy[i];
    }
    const double wh1 = sWH[c * NFTP + el * NFS + 1 * N + a];
    const double wh3 = sWH[c * NFTP + el * NFS + 3 * N + (N - 1 - a)];
    const double cx1 = gq[17] * (gq[10] * wh1) - tx1;
    const double cy1 = gq[17] * (gq[11] * wh1) - ty1;
    const double cx3 = -gq[19] * (gq[14] * wh3) - tx3;
    const double cy3 = -gq[19] * (gq[15] * wh3) - ty3;
    double* px = sPX + c * PS + el * ES + a * RS;
    double* py = sPY + c * PS + el * ES + a * RS;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double sx = 0.0, sy = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        sx += C.D[b * N + i] * wx[i];
        sy += C.D[b * N + i] * wy[i];
      }
      px[b] = (sx + C.lR[b] * cx1) - C.lL[b] * cx3;
      py[b] = (sy + C.lR[b] * cy1) - C.lL[b] * cy3;
    }
  }
  __syncthreads();
  // pass 2, columns: thread t = (b, el, c) finishes column b of both
  // gradient components and forms their traces on faces 0 (eL) and 2 (eR)
  // in sGF, summed in line_sum's order
  double* sGF = sm + L::F_GF;  // [2NW] padded face planes: gradient traces (CCW k)
  for (int t = t0; t < NLG; t += TH) {
    const int b = t / (E * NW), el = (t / NW) % E, c = t % NW;
    const double* gq = sG + el * 20;
    const Metric mt = metric(gq);
    const double* Wc = sW + c * PS + el * ES + b;
    double vx[N], vy[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double y = Wc[i * RS], eta = C.xg[i];
      vx[i] = -mt.J10(eta) * y;
      vy[i] = mt.J00(eta) * y;
    }
    double tx2 = 0.0, ty2 = 0.0, tx0 = 0.0, ty0 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      tx2 += C.eR[i] * vx[i];
      ty2 += C.eR[i] * vy[i];
      tx0 += C.eL[i] * vx[i];
      ty0 += C.eL[i] * vy[i];
    }
    const double wh2 = sWH[c * NFTP + el * NFS + 2 * N + (N - 1 - b)];
    const double wh0 = sWH[c * NFTP + el * NFS + 0 * N + b];
    const double cx2 = gq[18] * (gq[12] * wh2) - tx2;
    const double cy2 = gq[18] * (gq[13] * wh2) - ty2;
    const double cx0 = -gq[16] * (gq[8] * wh0) - tx0;
    const double cy0 = -gq[16] * (gq[9] * wh0) - ty0;
    const double xb = C.xg[b];
    const double j11b = mt.J11(xb), j01b = mt.J01(xb);
    double fx0 = 0.0, fy0 = 0.0, fx2 = 0.0, fy2 = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double dx = 0.0, dy = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        dx += C.D[a * N + i] * vx[i];
        dy += C.D[a * N + i] * vy[i];
      }
      double idet;
      if constexpr (PMGB_IDET_SMEM) {
        idet = sID[el * ES + a * RS + b];
      } else {
        const double xa = C.xg[a];
        idet = rcp(mt.J00(xa) * j11b - j01b * mt.J10(xa));
      }
      double* px = sPX + c * PS + el * ES + a * RS + b;
      double* py = sPY + c * PS + el * ES + a * RS + b;
      const double gxv = (((*px) + dx) + C.lR[a] * cx2 - C.lL[a] * cx0) * idet;
      const double gyv = (((*py) + dy) + C.lR[a] * cy2 - C.lL[a] * cy0) * idet;
      *px = gxv;
      *py = gyv;
      fx0 += C.eL[a] * gxv;
      fy0 += C.eL[a] * gyv;
      fx2 += C.eR[a] * gxv;
      fy2 += C.eR[a] * gyv;
    }
    const int s0 = el * NFS + 0 * N + b, s2 = el * NFS + 2 * N + (N - 1 - b);
    sGF[c * NFTP + s0] = fx0;
    sGF[(NW + c) * NFTP + s0] = fy0;
    sGF[c * NFTP + s2] = fx2;
    sGF[(NW + c) * NFTP + s2] = fy2;
  }
  __syncthreads();
  // pass 3, rows of the final gradients: traces on faces 1 (eR) and 3 (eL)
  for (int t = t0; t < NLG; t += TH) {
    const int c = t / (E * N), el = (t / N) % E, a = t % N;
    const double* gxr = sPX + c * PS + el * ES + a * RS;
    const double* gyr = sPY + c * PS + el * ES + a * RS;
    double fx1 = 0.0, fy1 = 0.0, fx3 = 0.0, fy3 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double x = gxr[i], y = gyr[i];
      fx1 += C.eR[i] * x;
      fy1 += C.eR[i] * y;
      fx3 += C.eL[i] * x;
      fy3 += C.eL[i] * y;
    }
    const int s1 = el * NFS + 1 * N + a, s3 = el * NFS + 3 * N + (N - 1 - a);
    sGF[c * NFTP + s1] = fx1;
    sGF[(NW + c) * NFTP + s1] = fy1;
    sGF[c * NFTP + s3] = fx3;
    sGF[(NW + c) * NFTP + s3] = fy3;
  }
  // point gradients to global: the CTA's 2NW padded planes are one
  // contiguous block of the [grid][2NW][PS] scratch (fr_grad_scratch_doubles)
  if (grad != nullptr) {
    constexpr int NB2 = NW * PS;  // double2 per block
    const double2* src = reinterpret_cast<const double2*>(sGR);
    double2* dst = reinterpret_cast<double2*>(grad + (int64_t)blockIdx.x * (2 * NW * PS));
    for (int i = t0; i < NB2; i += TH) dst[i] = src[i];
  }
  __syncthreads();
  // one-sided viscous normal flux on every own face point (spatial.py:456-464)
  auto face_fvn = [&](int el, int f, int k, const double* trv) {
    double gxv[NW], gyv[NW];
    const int slot = el * NFS + f * N + k;
#pragma unroll
    for (int c = 0; c < NW; ++c) {
      gxv[c] = sGF[c * NFTP + slot];
      gyv[c] = sGF[(NW + c) * NFTP + slot];
    }
    double fx[NV], fy[NV];
    visc_flux<KIND>(trv, gxv, gyv, ph, fx, fy);
    const double nx = sG[el * 20 + 8 + 2 * f], ny = sG[el * 20 + 9 + 2 * f];
    double o[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) o[v] = fx[v] * nx + fy[v] * ny;
    st_face<NV>(fvn + ((((int)e0 + el) * 4 + f) * N + k) * NV, o);
  };
  if constexpr (ONE_FACE) {
    // own trace still in registers from the prologue gather
    if (face_live) face_fvn(fel, ff, (t0 % NF) % N, tr);
  } else {
    for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
      const int el = t / NF, r = t % NF, f = r / N, k = r % N;
      if (e0 + el >= M) continue;
      double trv[NV];
      ld_face<NV>(qtr + ((((int)e0 + el) * 4 + f) * N + k) * NV, trv);
      face_fvn(el, f, k, trv);
    }
  }
}

// ---------------------------------------------------------------------------
// phase 3: common fluxes, volume fluxes, FR divergence, fused epilogue


// EK: compile-time epilogue mode as in k_assemble_async (-1 = runtime switch)
template <int P, int KIND, bool RKE = false, int EK = -1>
__global__ void __launch_bounds__(BC<P>::THREADS, EK >= 0 ? MinBlocks<P>::ASM_K : MinBlocks<P>::ASM)
k_assemble(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
           const double* __restrict__ fvn, const double* __restrict__ grad, const Epi ep,
           double* __restrict__ out, int* bad, Status* st) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW, NPT = L::NPT, NFT = L::NFT;
  constexpr bool VISC = KT<KIND>::VISC;
  if (blockIdx.x == 0 && threadIdx.x == 0) commit_status(bad, st);
  const Ops op = stage_ops<BC<P>::THREADS>(C, sm);
  double* sQ = sm + L::Q;
  double* sG = sm + L::G;
  double* sFC = sm + L::A_FC;
  double* sFT = sm + L::A_FT;
  double* sGT = sm + L::A_GT;
  double* sCF = sm + L::A_CF;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int64_t M = m.M;
  const Phys ph = phys_of(C);
  // Prologue: every global load of the kernel is issued before the first
  // barrier -- q / geometry into shared memory, the face gathers (own and
  // neighbour traces, one-sided viscous fluxes, the L side's normal) and
  // the point gradients into registers -- so their latencies overlap.
  static_assert(E * NF <= BC<P>::THREADS || P <= 2, "face prologue needs one face point per thread");
  constexpr bool ONE_FACE = (E * NF <= BC<P>::THREADS);
  const int t0 = threadIdx.x;
  load_points<P, NV>(q, e0, M, sQ);
  load_geom<P>(m.geom, e0, M, sG);
  double tr[NV], nb[NV], Fo[NV], Fn[NV], gx[NW], gy[NW];
  double nux = 0.0, nuy = 0.0;
  int2 lk = make_int2(-1, 0);
  bool face_live = false;
  int fel = 0, ff = 0, fk = 0;
  if constexpr (ONE_FACE) {
    if (t0 < E * NF) {
      fel = t0 / NF;
      const int r = t0 % NF;
      ff = r / N;
      fk = r % N;
      const int64_t e = e0 + fel;
      face_live = e < M;
      if (face_live) {
        lk = m.link[e * 4 + ff];
        const bool interior = lk.x >= 0;
        const int kk = lk_rev(lk.y) ? N - 1 - fk : fk;
        const int64_t own = ((e * 4 + ff) * N + fk) * NV;
        const int64_t nbi = interior ? (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV : own;
        ld_face<NV>(qtr + own, tr);
        ld_face<NV>(qtr + nbi, nb);
        if constexpr (VISC) {
          ld_face<NV>(fvn + own, Fo);
          ld_face<NV>(fvn + nbi, Fn);
        }
        if (interior && !lk_left(lk.y)) {
          const double* gn = m.geom + (int64_t)lk.x * 20 + 8 + 2 * lk_face(lk.y);
          nux = __ldg(gn);
          nuy = __ldg(gn + 1);
        }
      }
    }
  }
  if constexpr (VISC) {
    if (t0 < NPT) {
      const int el = t0 / NP, pt = t0 % NP;
      if (e0 + el < M) {
        // gradients in k_fvn's padded block layout
        const double* gs = grad + (int64_t)blockIdx.x * (2 * NW * L::PS) + L::pix(t0);
#pragma unroll
        for (int c = 0; c < NW; ++c) {
          gx[c] = __ldg(gs + c * L::PS);
          gy[c] = __ldg(gs + (NW + c) * L::PS);
        }
      } else {
#pragma unroll
        for (int c = 0; c < NW; ++c) gx[c] = gy[c] = 0.0;
      }
    }
  }
  __syncthreads();
  // common face fluxes: inviscid on the L side's normal (-F to R), viscous
  // 0.5 (fvn_own - fvn_nb), BR1 average (spatial.py:520-568).  Branch-free
  // across L/R sides: operands are selected, one Roe evaluation per thread.
  auto face_flux = [&](int t, int el, int f, int k, int2 lkk, double* tr_, double* nb_, const double* Fo_,
                       const double* Fn_, double nux_, double nuy_) {
    const double* gq = sG + el * 20;
    const double nx = gq[8 + 2 * f], ny = gq[9 + 2 * f];
    const bool interior = lkk.x >= 0;
    const bool left = !interior || lk_left(lkk.y);
    if (left) {
      nux_ = nx;
      nuy_ = ny;
    }
    if (!interior) ghost<KIND>(tr_, lk_tag(lkk.y), nx, ny, C.qinf, nb_);
    double qa[NV], qc[NV], F[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      qa[v] = left ? tr_[v] : nb_[v];
      qc[v] = left ? nb_[v] : tr_[v];
    }
    num_flux<KIND>(qa, qc, nux_, nuy_, ph, F);
#pragma unroll
    for (int v = 0; v < NV; ++v) F[v] = left ? F[v] : -F[v];
    if constexpr (VISC) {
      double Fv[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) Fv[v] = common_fv(ph, interior, left, Fo_[v], Fn_[v]);
      if (KT<KIND>::FLOW && !interior && lk_tag(lkk.y) == T_WALL_ADIABATIC) Fv[NV - 1] = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) F[v] = F[v] - Fv[v];
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) sFC[v * NFT + t] = F[v];
  };
  if constexpr (ONE_FACE) {
    if (face_live) face_flux(t0, fel, ff, fk, lk, tr, nb, Fo, Fn, nux, nuy);
  } else {
    for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
      const int el = t / NF, r = t % NF, f = r / N, k = r % N;
      const int64_t e = e0 + el;
      if (e >= M) continue;
      const int2 lkk = m.link[e * 4 + f];
      const bool interior = lkk.x >= 0;
      const int kk = lk_rev(lkk.y) ? N - 1 - k : k;
      const int64_t own = ((e * 4 + f) * N + k) * NV;
      const int64_t nbi = interior ? (((int64_t)lkk.x * 4 + lk_face(lkk.y)) * N + kk) * NV : own;
      double tr2[NV], nb2[NV], Fo2[NV], Fn2[NV];
      ld_face<NV>(qtr + own, tr2);
      ld_face<NV>(qtr + nbi, nb2);
      if constexpr (VISC) {
        ld_face<NV>(fvn + own, Fo2);
        ld_face<NV>(fvn + nbi, Fn2);
      }
      double nx2 = 0.0, ny2 = 0.0;
      if (interior && !lk_left(lkk.y)) {
        const double* gn = m.geom + (int64_t)lkk.x * 20 + 8 + 2 * lk_face(lkk.y);
        nx2 = __ldg(gn);
        ny2 = __ldg(gn + 1);
      }
      face_flux(t, el, f, k, lkk, tr2, nb2, Fo2, Fn2, nx2, ny2);
    }
  }
  // volume fluxes at the points: gradients come from k_fvn (same values
  // it used for the one-sided viscous fluxes)
  if (t0 < NPT) {
    const int el = t0 / NP, pt = t0 % NP, a = pt / N, b = pt % N;
    const Metric mt = metric(sG + el * 20);
    double qq[NV], Ft[NV], Gt[NV];
    gather_point<NV, NPT>(sQ, t0, qq);
    point_fluxes<P, KIND>(qq, gx, gy, ph, mt, op.xg[a], op.xg[b], Ft, Gt);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      sFT[v * NPT + t0] = Ft[v];
      sGT[v * NPT + t0] = Gt[v];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    if (e0 + el >= M) continue;
    double Fc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Fc[v] = sFC[v * NFT + t];
    flux_corrections<P, KIND>(op, sFT, sGT, sG + el * 20, Fc, sCF, el, f, k);
  }
  __syncthreads();
  if (t0 < NPT) {
    const int el = t0 / NP, pt = t0 % NP;
    const int64_t e = e0 + el;
    if (e < M) {
      const Metric mt = metric(sG + el * 20);
      double R[NV];
      divergence_at<P, KIND>(op, sFT, sGT, sCF, mt, el, pt / N, pt % N, R);
      const int64_t base = (e * NP + pt) * NV;
      double o[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if constexpr (EK >= 0 && !RKE) {
          Epi ek = ep;
          ek.mode = EK;   // constant: epi_apply's switch folds
          o[v] = epi_apply<false>(ek, base + v, R[v], sQ[v * NPT + t0]);
        } else {
          o[v] = epi_apply<RKE>(ep, base + v, R[v], sQ[v * NPT + t0]);
        }
      }
      st_face<NV>(out + base, o);
    }
  }
}

// cp.async (LDGSTS) helpers: 16-byte global->shared copies that do not
// stage through registers, so the issuing thread keeps running.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Phase 3, one face point per thread (p >= 3, 4 conserved variables):
// q and geometry go to shared memory by cp.async while the face threads
// gather their traces / fluxes and evaluate the common face fluxes straight
// from registers; the first barrier only guards the point stage.
// RKE: the RK-smoother stage epilogue is a separate instantiation (carrying
// its operand path in the R / Jv kernels measured 2.5 % on R at config 2)
// EK: the epilogue mode as a template constant for the hot modes (R, Jv,
// PTC Jv, defect, F; see run_residual), -1 = runtime switch for the rest.
// The plain-R instantiation carries no epilogue operands and gets its own
// register target (72 at p=4: 176.8 -> 162.4 us per R at config 2).
template <int P, int KIND, bool RKE = false, int EK = -1>
__global__ void __launch_bounds__(BC<P>::THREADS, EK == EPI_R ? MinBlocks<P>::ASM_R
                                                 : (RKE || EK >= 0 ? MinBlocks<P>::ASM_K : MinBlocks<P>::ASM))
k_assemble_async(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
                 const double* __restrict__ fvn, const double* __restrict__ grad, const Epi ep,
                 double* __restrict__ out, int* bad, Status* st, int q_dep) {
  extern __shared__ __align__(16) double sm[];
  using L = SL<P, KIND>;
  constexpr int TH = BC<P>::THREADS;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW, NPT = L::NPT, NFT = L::NFT;
  constexpr int PS = L::PS, ES = L::ES, RS = L::RS;
  constexpr bool VISC = KT<KIND>::VISC;
  static_assert(NV == 4 && E * NF <= TH, "async assemble: flow kinds, one face point per thread");
  double* sQA = sm + L::Q;  // AoS [E][NP][NV]
  double* sG = sm + L::G;
  double* sFC = sm + L::A_FC;
  double* sFT = sm + L::P_FT;  // [NV] padded point planes
  double* sGT = sm + L::P_GT;
  double* sID = sm + L::P_ID;  // 1/det J per point (point stage -> column pass)
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int64_t M = m.M;
  const int ne = (int)((M - e0) < E ? (M - e0) : E);
  const int t0 = threadIdx.x;
  // q_dep: q is k_trace's q + eps X (Jv forms): copied only after the wait
  auto copy_q = [&]() {
    const double* qs = q + e0 * NP * NV;
    for (int i = t0; i < E * NP * NV / 2; i += TH) cp_async16(sQA + 2 * i, qs + 2 * i, 2 * i < ne * NP * NV);
  };
  {
    if (!q_dep) copy_q();
    const double* gsrc = m.geom + e0 * 20;
    for (int i = t0; i < E * 10; i += TH) cp_async16(sG + 2 * i, gsrc + 2 * i, 2 * i < ne * 20);
    cp_async_commit();
  }
  // static mesh data of this thread's face point before the dependency wait
  const bool face_thread = t0 < E * NF && t0 / NF < ne;
  int2 lk = make_int2(-1, 0);
  double2 nu = make_double2(0.0, 0.0);
  if (face_thread) {
    const int fel = t0 / NF, f = (t0 % NF) / N;
    const int e = (int)e0 + fel;
    lk = m.link[e * 4 + f];
    const bool left = lk.x < 0 || lk_left(lk.y);
    const int gface = left ? e * 20 + 8 + 2 * f : lk.x * 20 + 8 + 2 * lk_face(lk.y);
    nu = __ldg(reinterpret_cast<const double2*>(m.geom + gface));
  }
  const Ops op = stage_ops<TH>(C, sm);
  const Phys ph = phys_of(C);
  pdl_wait();  // gradients / fvn from k_fvn, traces and status flags from k_trace
  if (q_dep) {
    copy_q();
    cp_async_commit();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) commit_status(bad, st);
  // point gradients into registers
  double gx[NW], gy[NW];
  if constexpr (VISC) {
#pragma unroll
    for (int c = 0; c < NW; ++c) gx[c] = gy[c] = 0.0;
    if (t0 < NPT) {
      const int el = t0 / NP, pt = t0 % NP;
      if (el < ne) {
        const double* gs = grad + (int64_t)blockIdx.x * (2 * NW * PS) + L::pix(t0);
#pragma unroll
        for (int c = 0; c < NW; ++c) {
          gx[c] = __ldg(gs + c * PS);
          gy[c] = __ldg(gs + (NW + c) * PS);
        }
      }
    }
  }
  // face threads: gathers and common face flux, no shared memory needed.
  // 32-bit element-relative offsets (host guarantees M*4*N*NV < 2^31); the
  // L/R operand order of the Roe flux is chosen by address, not by selects.
  if (face_thread) {
    const int fel = t0 / NF, r = t0 % NF, f = r / N, k = r % N;
    {
      const int e = (int)e0 + fel;
      const bool interior = lk.x >= 0;
      const bool left = !interior || lk_left(lk.y);
      const int kk = lk_rev(lk.y) ? N - 1 - k : k;
      const int own = ((e * 4 + f) * N + k) * NV;
      const int nbi = interior ? ((lk.x * 4 + lk_face(lk.y)) * N + kk) * NV : own;
      double qa[NV], qc[NV], Fo[NV], Fn[NV], F[NV];
      ld_face<NV>(qtr + (left ? own : nbi), qa);
      ld_face<NV>(qtr + (left ? nbi : own), qc);
      if constexpr (VISC) {
        ld_face<NV>(fvn + own, Fo);
        ld_face<NV>(fvn + nbi, Fn);
      }
      if (!interior) ghost<KIND>(qa, lk_tag(lk.y), nu.x, nu.y, C.qinf, qc);
      num_flux<KIND>(qa, qc, nu.x, nu.y, ph, F);
#pragma unroll
      for (int v = 0; v < NV; ++v) F[v] = left ? F[v] : -F[v];
      if constexpr (VISC) {
        double Fv[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) Fv[v] = common_fv(ph, interior, left, Fo[v], Fn[v]);
        if (!interior && lk_tag(lk.y) == T_WALL_ADIABATIC) Fv[NV - 1] = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] = F[v] - Fv[v];
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) sFC[v * NFT + t0] = F[v];
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (t0 < NPT) {
    const int el = t0 / NP, pt = t0 % NP, a = pt / N, b = pt % N;
    const Metric mt = metric(sG + el * 20);
    const double2 q01 = reinterpret_cast<const double2*>(sQA)[2 * t0];
    const double2 q23 = reinterpret_cast<const double2*>(sQA)[2 * t0 + 1];
    const double qq[NV] = {q01.x, q01.y, q23.x, q23.y};
    double Ft[NV], Gt[NV];
    point_fluxes<P, KIND>(qq, gx, gy, ph, mt, op.xg[a], op.xg[b], Ft, Gt);
    const int px0 = L::pix(t0);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      sFT[v * PS + px0] = Ft[v];
      sGT[v * PS + px0] = Gt[v];
    }
    if constexpr (PMGB_IDET_SMEM) {
      const double xa = op.xg[a], xb = op.xg[b];
      sID[px0] = rcp(mt.J00(xa) * mt.J11(xb) - mt.J01(xb) * mt.J10(xa));
    }
  }
  __syncthreads();
  // FR divergence by line threads (one per element, line, variable); the
  // operator coefficients are compile-time indexed kernel parameters
  // (constant bank), so the contractions read shared memory only for data.
  //   rows  : s[a][b] = sum_i D[b][i] Ft[a][i] + lR[b] c1[a] - lL[b] c3[a]
  //   cols  : R[a][b] = -(s[a][b] + sum_i D[a][i] Gt[i][b] + lR[a] c2[b] - lL[a] c0[b]) / det
  // with c_f = +-js_f Fc_f - (trace of Ft / Gt on face f)  (spatial.py:407-430)
  constexpr int NL = E * N * NV;
  if (t0 < NL) {
    const int el = t0 / (N * NV), r = t0 % (N * NV), a = r / NV, v = r % NV;
    double* rowp = sFT + v * PS + el * ES + a * RS;
    double x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = rowp[i];
    double t1 = 0.0, t3 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      t1 += C.eR[i] * x[i];
      t3 += C.eL[i] * x[i];
    }
    const double* gq = sG + el * 20;
    const double c1 = gq[17] * sFC[v * NFT + el * 4 * N + 1 * N + a] - t1;
    const double c3 = -gq[19] * sFC[v * NFT + el * 4 * N + 3 * N + (N - 1 - a)] - t3;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double sb = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) sb += C.D[b * N + i] * x[i];
      rowp[b] = (sb + C.lR[b] * c1) - C.lL[b] * c3;  // in place: this thread owns row a
    }
  }
  __syncthreads();
  if (t0 < NL) {
    const int el = t0 / (N * NV), r = t0 % (N * NV), b = r / NV, v = r % NV;
    if (el < ne) {
      const double* colp = sGT + v * PS + el * ES + b;
      double y[N];
#pragma unroll
      for (int i = 0; i < N; ++i) y[i] = colp[i * RS];
      double t2 = 0.0, t0f = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        t2 += C.eR[i] * y[i];
        t0f += C.eL[i] * y[i];
      }
      const double* gq = sG + el * 20;
      const Metric mt = metric(gq);
      const double c2 = gq[18] * sFC[v * NFT + el * 4 * N + 2 * N + (N - 1 - b)] - t2;
      const double c0 = -gq[16] * sFC[v * NFT + el * 4 * N + 0 * N + b] - t0f;
      const double xb = C.xg[b];
      const double j11 = mt.J11(xb), j01 = mt.J01(xb);
      const int64_t e = e0 + el;
      double o1[N], o2[N], o3[N];
      if constexpr (EK != EPI_R) {
#pragma unroll
        for (int a = 0; a < N; ++a) epi_load_k<RKE ? EPI_RK : EK>(ep, (e * NP + a * N + b) * NV + v, o1[a], o2[a], o3[a]);
      }
      const double ce = RKE ? epi_rk_coef(ep, e) : 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double ta = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) ta += C.D[a * N + i] * y[i];
        double idet;
        if constexpr (PMGB_IDET_SMEM) {
          idet = sID[el * ES + a * RS + b];
        } else {
          const double xa = C.xg[a];
          idet = rcp(mt.J00(xa) * j11 - j01 * mt.J10(xa));
        }
        double d = sFT[v * PS + el * ES + a * RS + b] + ta;
        d = (d + C.lR[a] * c2) - C.lL[a] * c0;
        const double R = -(d * idet);
        const int pt = a * N + b;
        const int64_t gi = (e * NP + pt) * NV + v;
        const double qv = sQA[(el * NP + pt) * NV + v];
        if constexpr (EK == EPI_R)
          out[gi] = R;
        else
          out[gi] = RKE ? epi_rk(ep, ce, R, qv, o1[a], o2[a], o3[a]) : epi_pre_k<EK>(ep, R, qv, o1[a], o2[a], o3[a]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// element-local residual with frozen neighbour data (spatial.py:768-853)
//
// Slot s of the CTA holds one (element, state) instance in the Q planes;
// neighbours enter only through the frozen traces qtr and one-sided
// viscous fluxes fvn of the linearisation state.  Fluxes are evaluated on
// the element's own normal (the reference's local path).  Leaves the
// local residual of point thread t in R (valid when t < NPT and the slot
// is live).

// OV: face ov_face of every slot takes its neighbour data from the
// per-slot records in shared memory (sm + OVQ / OVF, aligned to the slot's
// own face points) instead of the frozen buffers -- the reference's
// element_residual face_override (spatial.py:787-790).
template <int P, int KIND, bool OV = false>
__device__ __forceinline__ void local_pipeline(const FrConst& C, const FrMesh& m, const Ops& op, double* sm,
                                               const int64_t* slot_elem, const double* __restrict__ qtr,
                                               const double* __restrict__ fvn, double* R, int ov_face = -1) {
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW, NPT = L::NPT, NFT = L::NFT;
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
    if (t0 < NPT) {
      double qq[NV], w[NW];
      gather_point<NV, NPT>(sQ, t0, qq);
      grad_vars<KIND>(qq, ph.gamma, w);
#pragma unroll
      for (int c = 0; c < NW; ++c) sW[c * NPT + t0] = w[c];
    }
  }
  for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = slot_elem[el];
    if (e < 0) continue;
    const int2 lk = m.link[e * 4 + f];
    const double* gq = sG + el * 20;
    const double nx = gq[8 + 2 * f], ny = gq[9 + 2 * f];
    double tr[NV], nb[NV], F[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = line_sum<N>(op, sQ + v * NPT + el * NP, f, k);
    if (OV && f == ov_face) {
#pragma unroll
      for (int v = 0; v < NV; ++v) nb[v] = sm[L::OVQ + (el * N + k) * NV + v];
    } else if (lk.x >= 0) {
      const int kk = lk_rev(lk.y) ? N - 1 - k : k;
      ld_face<NV>(qtr + (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV, nb);
    } else {
      ghost<KIND>(tr, lk_tag(lk.y), nx, ny, C.qinf, nb);
    }
    num_flux<KIND>(tr, nb, nx, ny, ph, F);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      sFC[v * NFT + t] = F[v];
      sTR[v * NFT + t] = tr[v];
    }
    if constexpr (VISC) {
      double wa[NW], wc[NW];
      grad_vars<KIND>(tr, ph.gamma, wa);
      grad_vars<KIND>(nb, ph.gamma, wc);
      if (lk.x < 0) ghost_w<KIND>(ph, lk_tag(lk.y), wa, wc);
      const bool inter = lk.x >= 0, lft = inter && lk_left(lk.y);
#pragma unroll
      for (int c = 0; c < NW; ++c) sWH[c * NFT + t] = common_w(ph, inter, lft, wa[c], wc[c]);
    }
  }
  __syncthreads();
  if constexpr (VISC) {
    for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
      const int el = t / NF, r = t % NF, f = r / N, k = r % N;
      if (slot_elem[el] < 0) continue;
      grad_corrections<P, KIND>(op, sW, sG + el * 20, sWH, sCG, el, f, k);
    }
    __syncthreads();
  }
  if (t0 < NPT) {
    const int el = t0 / NP, pt = t0 % NP, a = pt / N, b = pt % N;
    double gx[NW], gy[NW];
    if constexpr (VISC) {
      gradient_at<P, KIND>(op, sW, sG + el * 20, sCG, el, a, b, gx, gy);
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        sGR[c * NPT + t0] = gx[c];
        sGR[(NW + c) * NPT + t0] = gy[c];
      }
    }
    const Metric mt = metric(sG + el * 20);
    double qq[NV], Ft[NV], Gt[NV];
    gather_point<NV, NPT>(sQ, t0, qq);
    point_fluxes<P, KIND>(qq, gx, gy, ph, mt, op.xg[a], op.xg[b], Ft, Gt);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      sFT[v * NPT + t0] = Ft[v];
      sGT[v * NPT + t0] = Gt[v];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = slot_elem[el];
    if (e < 0) continue;
    double Fc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Fc[v] = sFC[v * NFT + t];
    if constexpr (VISC) {
      double gx[NW], gy[NW];
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        gx[c] = line_sum<N>(op, sGR + c * NPT + el * NP, f, k);
        gy[c] = line_sum<N>(op, sGR + (NW + c) * NPT + el * NP, f, k);
      }
      double tr[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) tr[v] = sTR[v * NFT + t];
      double fx[NV], fy[NV];
      visc_flux<KIND>(tr, gx, gy, ph, fx, fy);
      const double nx = sG[el * 20 + 8 + 2 * f], ny = sG[el * 20 + 9 + 2 * f];
      const int2 lk = m.link[e * 4 + f];
      double Fv[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) Fv[v] = fx[v] * nx + fy[v] * ny;
      if (OV && f == ov_face) {
        const bool lft = lk_left(lk.y);
#pragma unroll
        for (int v = 0; v < NV; ++v) Fv[v] = common_fv(ph, true, lft, Fv[v], sm[L::OVF + (el * N + k) * NV + v]);
      } else if (lk.x >= 0) {
        const int kk = lk_rev(lk.y) ? N - 1 - k : k;
        const bool lft = lk_left(lk.y);
        double Fn[NV];
        ld_face<NV>(fvn + (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV, Fn);
#pragma unroll
        for (int v = 0; v < NV; ++v) Fv[v] = common_fv(ph, true, lft, Fv[v], Fn[v]);
      } else if (KT<KIND>::FLOW && lk_tag(lk.y) == T_WALL_ADIABATIC) {
        Fv[NV - 1] = 0.0;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) Fc[v] = Fc[v] - Fv[v];
    }
    // CF aliases CG, whose last readers (gradient_at) finished before the
    // previous barrier
    flux_corrections<P, KIND>(op, sFT, sGT, sG + el * 20, Fc, sCF, el, f, k);
  }
  __syncthreads();
  if (t0 < NPT) {
    const int el = t0 / NP, pt = t0 % NP;
    if (slot_elem[el] >= 0) {
      const Metric mt = metric(sG + el * 20);
      divergence_at<P, KIND>(op, sFT, sGT, sCF, mt, el, pt / N, pt % N, R);
    }
  }
}

// batched element-local residual: instance b = (elems[b], Q[b])
template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS, MinBlocks<P>::ASM)
k_local(const FrConst C, const FrMesh m, const int64_t* __restrict__ elems, int64_t B,
        const double* __restrict__ Q, const double* __restrict__ qtr, const double* __restrict__ fvn,
        double* __restrict__ out) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB, NV = KT<KIND>::NV;
  __shared__ int64_t slot[E];
  const Ops op = stage_ops<BC<P>::THREADS>(C, sm);
  const int64_t b0 = (int64_t)blockIdx.x * E;
  for (int s = threadIdx.x; s < E; s += BC<P>::THREADS) slot[s] = (b0 + s < B) ? elems[b0 + s] : -1;
  load_points<P, NV>(Q, b0, B, sm + L::Q);
  __syncthreads();
  for (int i = threadIdx.x; i < E * 20; i += BC<P>::THREADS) {
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
__global__ void __launch_bounds__(BC<P>::THREADS, MinBlocks<P>::BLK)
k_blocks(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
         const double* __restrict__ fvn, double shift, double eps, double* __restrict__ BT,
         const int* __restrict__ out_slot) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB, NV = KT<KIND>::NV, NPT = L::NPT;
  constexpr int SZ = NP * NV;
  __shared__ int64_t slot[E];
  const Ops op = stage_ops<BC<P>::THREADS>(C, sm);
  const int64_t e = blockIdx.x;
  double* sQ = sm + L::Q;
  double* sR0 = sm + L::R0;
  const double* qe = q + e * SZ;
  const int t0 = threadIdx.x;
  double* BTe = BT + (out_slot ? (int64_t)out_slot[e] : e) * (int64_t)SZ * SZ;
  for (int i = threadIdx.x; i < E * 20; i += BC<P>::THREADS) sm[L::G + i] = __ldg(m.geom + e * 20 + i % 20);
  for (int c0 = 0; c0 <= SZ; c0 += E) {
    __syncthreads();
    for (int s = threadIdx.x; s < E; s += BC<P>::THREADS) slot[s] = (c0 + s <= SZ) ? e : -1;
    for (int i = threadIdx.x; i < E * SZ; i += BC<P>::THREADS) {
      const int s = i / SZ, d = i % SZ, c = c0 + s;
      const double v = __ldg(qe + d);
      sQ[(d % NV) * NPT + s * NP + d / NV] = (c >= 1 && d == c - 1) ? v + eps : v;
    }
    __syncthreads();
    double R[NV];
    local_pipeline<P, KIND>(C, m, op, sm, slot, qtr, fvn, R);
    const int s = t0 / NP, pt = t0 % NP, c = c0 + s;
    if (c0 == 0 && t0 < NP) {
#pragma unroll
      for (int v = 0; v < NV; ++v) sR0[pt * NV + v] = R[v];
    }
    __syncthreads();
    if (t0 < NPT && c >= 1 && c <= SZ) {
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
// neighbour face records and FD coupling blocks (spatial.py:855-903,
// newton_krylov.py:254-311)
//
// record_pipeline: the slots hold (perturbed) states of the neighbour nb of
// element e across e's face f; it runs nb's own trace / BR1 / gradient
// pipeline with nb's other neighbours frozen and leaves, aligned to e's face
// points, nb's trace (OVQ) and one-sided viscous normal flux (OVF) on the
// shared face fnb.

template <int P, int KIND>
__device__ __forceinline__ void record_pipeline(const FrConst& C, const FrMesh& m, const Ops& op, double* sm,
                                                const int64_t* slot_elem, const double* __restrict__ qtr,
                                                int fnb, bool rev) {
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, NP = BC<P>::NP, NF = BC<P>::NF, E = BC<P>::EPB;
  constexpr int NV = KT<KIND>::NV, NW = KT<KIND>::NW, NPT = L::NPT, NFT = L::NFT;
  constexpr bool VISC = KT<KIND>::VISC;
  double* sQ = sm + L::Q;
  double* sG = sm + L::G;
  double* sW = sm + L::W;
  double* sWH = sm + L::WH;
  double* sCG = sm + L::CG;
  double* sGR = sm + L::GR;
  double* sTR = sm + L::TR;
  const Phys ph = phys_of(C);
  const int t0 = threadIdx.x;
  if constexpr (VISC) {
    if (t0 < NPT) {
      double qq[NV], w[NW];
      gather_point<NV, NPT>(sQ, t0, qq);
      grad_vars<KIND>(qq, ph.gamma, w);
#pragma unroll
      for (int c = 0; c < NW; ++c) sW[c * NPT + t0] = w[c];
    }
  }
  for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
    const int el = t / NF, r = t % NF, f = r / N, k = r % N;
    const int64_t e = slot_elem[el];
    if (e < 0) continue;
    double tr[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) tr[v] = line_sum<N>(op, sQ + v * NPT + el * NP, f, k);
    if (f == fnb) {
      const int ke = rev ? N - 1 - k : k;
#pragma unroll
      for (int v = 0; v < NV; ++v) sm[L::OVQ + (el * N + ke) * NV + v] = tr[v];
    }
    if constexpr (VISC) {
      const int2 lk = m.link[e * 4 + f];
      const double* gq = sG + el * 20;
      double nb[NV];
      if (lk.x >= 0) {
        const int kk = lk_rev(lk.y) ? N - 1 - k : k;
        ld_face<NV>(qtr + (((int64_t)lk.x * 4 + lk_face(lk.y)) * N + kk) * NV, nb);
      } else {
        ghost<KIND>(tr, lk_tag(lk.y), gq[8 + 2 * f], gq[9 + 2 * f], C.qinf, nb);
      }
      double wa[NW], wc[NW];
      grad_vars<KIND>(tr, ph.gamma, wa);
      grad_vars<KIND>(nb, ph.gamma, wc);
      if (lk.x < 0) ghost_w<KIND>(ph, lk_tag(lk.y), wa, wc);
      const bool inter = lk.x >= 0, lft = inter && lk_left(lk.y);
#pragma unroll
      for (int c = 0; c < NW; ++c) sWH[c * NFT + t] = common_w(ph, inter, lft, wa[c], wc[c]);
#pragma unroll
      for (int v = 0; v < NV; ++v) sTR[v * NFT + t] = tr[v];
    }
  }
  if constexpr (VISC) {
    __syncthreads();
    for (int t = threadIdx.x; t < E * NF; t += BC<P>::THREADS) {
      const int el = t / NF, r = t % NF, f = r / N, k = r % N;
      if (slot_elem[el] < 0) continue;
      grad_corrections<P, KIND>(op, sW, sG + el * 20, sWH, sCG, el, f, k);
    }
    __syncthreads();
    if (t0 < NPT) {
      const int el = t0 / NP, pt = t0 % NP;
      double gx[NW], gy[NW];
      gradient_at<P, KIND>(op, sW, sG + el * 20, sCG, el, pt / N, pt % N, gx, gy);
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        sGR[c * NPT + t0] = gx[c];
        sGR[(NW + c) * NPT + t0] = gy[c];
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < E * N; t += BC<P>::THREADS) {
      const int el = t / N, k = t % N;
      if (slot_elem[el] < 0) continue;
      const int fi = el * NF + fnb * N + k;
      double gx[NW], gy[NW], tr[NV], fx[NV], fy[NV];
#pragma unroll
      for (int c = 0; c < NW; ++c) {
        gx[c] = line_sum<N>(op, sGR + c * NPT + el * NP, fnb, k);
        gy[c] = line_sum<N>(op, sGR + (NW + c) * NPT + el * NP, fnb, k);
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) tr[v] = sTR[v * NFT + fi];
      visc_flux<KIND>(tr, gx, gy, ph, fx, fy);
      const double nx = sG[el * 20 + 8 + 2 * fnb], ny = sG[el * 20 + 9 + 2 * fnb];
      const int ke = rev ? N - 1 - k : k;
#pragma unroll
      for (int v = 0; v < NV; ++v) sm[L::OVF + (el * N + ke) * NV + v] = fx[v] * nx + fy[v] * ny;
    }
  }
}

// One CTA per (element e, face f) coupling: column c of -dR_e/dq_nb from
// instance c (nb's state with DoF c-1 raised by eps; instance 0 is the base).
// Output column-major into the block slot (BT[c][r] = B[r][c]); pair_add
// accumulates onto what an earlier wave (or the element block) wrote there (periodic pairs meeting
// through two faces, newton_krylov.py:307-310).
template <int P, int KIND>
__global__ void __launch_bounds__(BC<P>::THREADS)
k_coupling(const FrConst C, const FrMesh m, const double* __restrict__ q, const double* __restrict__ qtr,
           const double* __restrict__ fvn, double eps, const int* __restrict__ pair_e,
           const signed char* __restrict__ pair_f, const int* __restrict__ pair_slot,
           const signed char* __restrict__ pair_add, double* __restrict__ blocks) {
  extern __shared__ double sm[];
  using L = SL<P, KIND>;
  constexpr int NP = BC<P>::NP, E = BC<P>::EPB, NV = KT<KIND>::NV, NPT = L::NPT;
  constexpr int SZ = NP * NV;
  __shared__ int64_t slot[E];
  const Ops op = stage_ops<BC<P>::THREADS>(C, sm);
  const int64_t e = pair_e[blockIdx.x];
  const int f = pair_f[blockIdx.x];
  const int2 lk = m.link[e * 4 + f];
  const int64_t nb = lk.x;
  const int fnb = lk_face(lk.y);
  const bool rev = lk_rev(lk.y);
  double* sQ = sm + L::Q;
  double* sR0 = sm + L::R0;
  double* out = blocks + (int64_t)pair_slot[blockIdx.x] * SZ * SZ;
  const bool add = pair_add[blockIdx.x] != 0;
  const int t0 = threadIdx.x;
  for (int c0 = 0; c0 <= SZ; c0 += E) {
    // neighbour records for instances c0 .. c0+E-1
    __syncthreads();
    for (int i = threadIdx.x; i < E * 20; i += BC<P>::THREADS) sm[L::G + i] = __ldg(m.geom + nb * 20 + i % 20);
    for (int s = threadIdx.x; s < E; s += BC<P>::THREADS) slot[s] = (c0 + s <= SZ) ? nb : -1;
    for (int i = threadIdx.x; i < E * SZ; i += BC<P>::THREADS) {
      const int s = i / SZ, d = i % SZ, c = c0 + s;
      const double v = __ldg(q + nb * SZ + d);
      sQ[(d % NV) * NPT + s * NP + d / NV] = (c >= 1 && d == c - 1) ? v + eps : v;
    }
    __syncthreads();
    record_pipeline<P, KIND>(C, m, op, sm, slot, qtr, fnb, rev);
    // element e (unperturbed) with face f overridden by the records
    __syncthreads();
    for (int i = threadIdx.x; i < E * 20; i += BC<P>::THREADS) sm[L::G + i] = __ldg(m.geom + e * 20 + i % 20);
    for (int s = threadIdx.x; s < E; s += BC<P>::THREADS) slot[s] = (c0 + s <= SZ) ? e : -1;
    for (int i = threadIdx.x; i < E * SZ; i += BC<P>::THREADS) {
      const int s = i / SZ, d = i % SZ;
      sQ[(d % NV) * NPT + s * NP + d / NV] = __ldg(q + e * SZ + d);
    }
    __syncthreads();
    double R[NV];
    local_pipeline<P, KIND, true>(C, m, op, sm, slot, qtr, fvn, R, f);
    const int s = t0 / NP, pt = t0 % NP, c = c0 + s;
    if (c0 == 0 && t0 < NP) {
#pragma unroll
      for (int v = 0; v < NV; ++v) sR0[pt * NV + v] = R[v];
    }
    __syncthreads();
    if (t0 < NPT && c >= 1 && c <= SZ) {
      double* col = out + (int64_t)(c - 1) * SZ;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int i = pt * NV + v;
        const double val = -(R[v] - sR0[i]) / eps;
        col[i] = add ? col[i] + val : val;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// wall forces (compute_forces, spatial.py:633-695): thread per wall
// (element, face); pressure p n minus the viscous traction tau n at every
// face point, from the traces of q (qtr) and of k_fvn's BR1 point
// gradients (padded block scratch), weighted by w_k * face_jac.  One
// 2-vector per face; the host sums them in face order.
struct FaceWeights {
  double w[6];
};

template <int P, int KIND>
__global__ void __launch_bounds__(128)
k_wall_forces(const FrConst C, const FrMesh m, const double* __restrict__ qtr, const double* __restrict__ grad,
              const int* __restrict__ wall_e, const signed char* __restrict__ wall_f, int64_t nwall,
              const FaceWeights fw, double* __restrict__ out) {
  using L = SL<P, KIND>;
  constexpr int N = BC<P>::N, E = BC<P>::EPB, NW = KT<KIND>::NW;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nwall) return;
  const int64_t e = wall_e[t];
  const int f = wall_f[t];
  const double* g = m.geom + e * 20;
  const double nx = g[8 + 2 * f], ny = g[9 + 2 * f], js = g[16 + f];
  const double* eline = (f == 0 || f == 3) ? C.eL : C.eR;
  const int64_t blk = e / E;
  const int el = (int)(e - blk * E);
  const double* gb = grad + blk * (2 * NW * L::PS);
  double Fx = 0.0, Fy = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double q[4];
    ld_face<4>(qtr + ((e * 4 + f) * N + k) * 4, q);
    double r, ir, u, v, p;
    prim(q, C.gamma, r, ir, u, v, p);
    double cx = p * nx, cy = p * ny;
    if constexpr (KT<KIND>::VISC) {
      // face line of (f, k): points base + i * stride (face_line)
      const int base = f == 0 ? k : f == 1 ? k * N : f == 2 ? (N - 1 - k) : (N - 1 - k) * N;
      const int stride = (f == 0 || f == 2) ? N : 1;
      double gt[2 * NW];
#pragma unroll
      for (int c = 0; c < 2 * NW; ++c) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const int pt = base + i * stride;
          s += eline[i] * __ldg(gb + c * L::PS + L::pix(el, pt / N, pt % N));
        }
        gt[c] = s;
      }
      const double ux = gt[0], vx = gt[1], uy = gt[NW + 0], vy = gt[NW + 1];
      const double div = ux + vy;
      const double txx = C.mu * (2 * ux - (2.0 / 3.0) * div);
      const double tyy = C.mu * (2 * vy - (2.0 / 3.0) * div);
      const double txy = C.mu * (uy + vx);
      cx = cx - (txx * nx + txy * ny);
      cy = cy - (txy * nx + tyy * ny);
    }
    Fx += fw.w[k] * (js * cx);
    Fy += fw.w[k] * (js * cy);
  }
  out[2 * t] = Fx;
  out[2 * t + 1] = Fy;
}

// ---------------------------------------------------------------------------
// host-side dispatch

// ---------------------------------------------------------------------------
// RK smoother: per-element spectral-radius estimate (oracle:
// solver_oracle.rk_spectral_radius).  One warp per element, lanes over the
// points; max / min are order-independent, so the result is deterministic.
__global__ void __launch_bounds__(256)
k_rk_lambda(const FrConst C, const FrMesh m, int p, int kind, const double* __restrict__ q, double adv,
            double* __restrict__ lam) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= m.M) return;
  const int n = p + 1, NP = n * n;
  double amax = 0.0, rmin = INFINITY;
  if (kind == K_ADV || kind == K_ADVD) {
    amax = sqrt(C.adv_x * C.adv_x + C.adv_y * C.adv_y);
  } else {
    const double g = C.gamma;
    for (int t = lane; t < NP; t += 32) {
      const double* qp = q + (e * NP + t) * 4;
      const double r = qp[0];
      const double u = qp[1] / r, v = qp[2] / r;
      const double pr = (g - 1.0) * (qp[3] - 0.5 * r * (u * u + v * v));
      const double a = sqrt(u * u + v * v) + sqrt(g * pr / r);
      amax = fmax(amax, a);
      rmin = fmin(rmin, r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      rmin = fmin(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
    }
  }
  if (lane != 0) return;
  const double* gq = m.geom + e * 20;
  const double a0 = gq[0], b0 = gq[2], c0 = gq[4], d0 = gq[6];
  const double Lx = 2.0 * sqrt(a0 * a0 + b0 * b0);
  const double Ly = 2.0 * sqrt(c0 * c0 + d0 * d0);
  const double h = 4.0 * fabs(a0 * d0 - c0 * b0) / fmax(Lx, Ly);
  double nu = 0.0;
  if (kind == K_NS) nu = fmax(4.0 / 3.0 * C.mu, C.kappa * (C.gamma - 1.0)) / rmin;
  else if (kind == K_ADVD) nu = C.diff;
  const double pp = (double)(n * n) * (double)(n * n);
  lam[e] = adv * amax / h + pp * nu / (h * h);
}

int launch_rk_lambda(const DiscDev& d, const double* q, double adv, double* lam, cudaStream_t st) {
  if (d.M == 0) return 0;
  const unsigned grid = (unsigned)((d.M * 32 + 255) / 256);
  k_rk_lambda<<<grid, 256, 0, st>>>(d.C, d.mesh, d.p, d.kind, q, adv, lam);
  return (int)cudaGetLastError();
}

static __device__ int g_bad[2] = {INT_MAX, INT_MAX};
static __device__ Status g_status = {0, 0, 0};

// launch with programmatic stream serialization (PDL) enabled
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), unsigned grid, int threads, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// PMGB_EPI_SPECIALIZE=0 forces the runtime-switch instantiation (A/B)
static bool epi_specialize() {
  static const bool on = [] {
    const char* v = std::getenv("PMGB_EPI_SPECIALIZE");
    return v == nullptr || v[0] != '0';
  }();
  return on;
}

using AsmAsyncFn = void (*)(const FrConst, const FrMesh, const double*, const double*, const double*, const double*,
                            const Epi, double*, int*, Status*, int);

using AsmFn = void (*)(const FrConst, const FrMesh, const double*, const double*, const double*, const double*,
                       const Epi, double*, int*, Status*);

template <int P, int KIND>
static AsmFn asm_for(int mode) {
  if (!epi_specialize()) return k_assemble<P, KIND>;
  switch (mode) {
    case EPI_R: return k_assemble<P, KIND, false, EPI_R>;
    case EPI_JV: return k_assemble<P, KIND, false, EPI_JV>;
    case EPI_STAGE_JV: return k_assemble<P, KIND, false, EPI_STAGE_JV>;
    case EPI_DEFECT: return k_assemble<P, KIND, false, EPI_DEFECT>;
    case EPI_F: return k_assemble<P, KIND, false, EPI_F>;
  }
  return k_assemble<P, KIND>;
}

template <int P, int KIND>
static AsmAsyncFn asm_async_for(int mode) {
  if (mode == EPI_RK) return k_assemble_async<P, KIND, true>;
  if (!epi_specialize()) return k_assemble_async<P, KIND, false>;
  switch (mode) {
    case EPI_R: return k_assemble_async<P, KIND, false, EPI_R>;
    case EPI_JV: return k_assemble_async<P, KIND, false, EPI_JV>;
    case EPI_STAGE_JV: return k_assemble_async<P, KIND, false, EPI_STAGE_JV>;
    case EPI_DEFECT: return k_assemble_async<P, KIND, false, EPI_DEFECT>;
    case EPI_F: return k_assemble_async<P, KIND, false, EPI_F>;
  }
  return k_assemble_async<P, KIND, false>;
}

template <int P, int KIND>
static int run_residual(const DiscDev& d, const double* q, const double* X, double eps, const Epi& epi,
                        double* out, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB, TH = BC<P>::THREADS;
  static std::atomic<unsigned long long> attr_seen{0};
  once_per_device(attr_seen, [&] {
    cudaFuncSetAttribute(k_trace<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_TRACE);
    cudaFuncSetAttribute(k_fvn<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_FVN);
    cudaFuncSetAttribute(k_assemble<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_ASM);
    cudaFuncSetAttribute(k_assemble<P, KIND, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_ASM);
    for (int md : {(int)EPI_R, (int)EPI_JV, (int)EPI_STAGE_JV, (int)EPI_DEFECT, (int)EPI_F})
      cudaFuncSetAttribute(asm_for<P, KIND>(md), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_ASM);
    if constexpr (KT<KIND>::NV == 4 && E * BC<P>::NF <= TH) {
      cudaFuncSetAttribute(k_assemble_async<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_ASYNC);
      for (int md : {(int)EPI_R, (int)EPI_JV, (int)EPI_STAGE_JV, (int)EPI_DEFECT, (int)EPI_F})
        cudaFuncSetAttribute(asm_async_for<P, KIND>(md), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)L::BYTES_ASYNC);
      cudaFuncSetAttribute(k_assemble_async<P, KIND, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)L::BYTES_ASYNC);
    }
  });
  int* bad = nullptr;
  Status* stp = nullptr;
  cudaGetSymbolAddress((void**)&bad, g_bad);
  cudaGetSymbolAddress((void**)&stp, g_status);
  if (d.has_rect && rect_supported(P, KIND))
    return launch_residual_rect(d.rect, d, q, X, eps, epi, out, bad, stp, st);
  const unsigned grid = (unsigned)((d.M + E - 1) / E);
  const double* qq = q;
  if (X != nullptr) qq = d.qp;
  if constexpr (KT<KIND>::FLOW) {
    const unsigned gl = (unsigned)((d.M * 2 * (P + 1) + 127) / 128);
    if (X != nullptr)
      k_trace_lines<P, KIND, true><<<gl, 128, 0, st>>>(d.C, d.mesh, q, X, eps, d.qp, d.qtr, bad);
    else
      k_trace_lines<P, KIND, false><<<gl, 128, 0, st>>>(d.C, d.mesh, q, X, eps, d.qp, d.qtr, bad);
  } else {
    k_trace<P, KIND><<<grid, TH, L::BYTES_TRACE, st>>>(d.C, d.mesh, q, X, eps, d.qp, d.qtr, bad);
  }
  const int q_dep = X != nullptr;
  if (KT<KIND>::VISC) launch_pdl(k_fvn<P, KIND>, grid, TH, L::BYTES_FVN, st, d.C, d.mesh, qq, (const double*)d.qtr,
                                 d.fvn, d.grad, q_dep);
  const bool rk = epi.mode == EPI_RK;
  if constexpr (KT<KIND>::NV == 4 && E * BC<P>::NF <= TH)
    launch_pdl(asm_async_for<P, KIND>(epi.mode), grid, TH, L::BYTES_ASYNC, st, d.C, d.mesh, qq,
               (const double*)d.qtr, (const double*)d.fvn, (const double*)d.grad, epi, out, bad, stp, q_dep);
  else if (rk)
    k_assemble<P, KIND, true><<<grid, TH, L::BYTES_ASM, st>>>(d.C, d.mesh, qq, d.qtr, d.fvn, d.grad, epi, out, bad,
                                                               stp);
  else
    asm_for<P, KIND>(epi.mode)<<<grid, TH, L::BYTES_ASM, st>>>(d.C, d.mesh, qq, d.qtr, d.fvn, d.grad, epi, out, bad,
                                                              stp);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_freeze(const DiscDev& d, const double* q, double* qtr, double* fvn, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB, TH = BC<P>::THREADS;
  static std::atomic<unsigned long long> attr_seen{0};
  once_per_device(attr_seen, [&] {
    cudaFuncSetAttribute(k_trace<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_TRACE);
    cudaFuncSetAttribute(k_fvn<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_FVN);
  });
  const unsigned grid = (unsigned)((d.M + E - 1) / E);
  if constexpr (KT<KIND>::FLOW) {
    const unsigned gl = (unsigned)((d.M * 2 * (P + 1) + 127) / 128);
    k_trace_lines<P, KIND><<<gl, 128, 0, st>>>(d.C, d.mesh, q, nullptr, 0.0, nullptr, qtr, nullptr);
  } else {
    k_trace<P, KIND><<<grid, TH, L::BYTES_TRACE, st>>>(d.C, d.mesh, q, nullptr, 0.0, nullptr, qtr, nullptr);
  }
  if (KT<KIND>::VISC) k_fvn<P, KIND><<<grid, TH, L::BYTES_FVN, st>>>(d.C, d.mesh, q, qtr, fvn, nullptr, 0);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_local(const DiscDev& d, const int64_t* elems, int64_t B, const double* Q, const double* qtr,
                     const double* fvn, double* out, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB, TH = BC<P>::THREADS;
  static std::atomic<unsigned long long> attr_seen{0};
  once_per_device(attr_seen, [&] {
    cudaFuncSetAttribute(k_local<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_LOCAL);
  });
  if (B <= 0) return 0;
  const unsigned grid = (unsigned)((B + E - 1) / E);
  k_local<P, KIND><<<grid, TH, L::BYTES_LOCAL, st>>>(d.C, d.mesh, elems, B, Q, qtr, fvn, out);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_blocks(const DiscDev& d, const double* q, const double* qtr, const double* fvn, double shift,
                      double eps, double* BT, const int* out_slot, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int TH = BC<P>::THREADS;
  static std::atomic<unsigned long long> attr_seen{0};
  once_per_device(attr_seen, [&] {
    cudaFuncSetAttribute(k_blocks<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_LOCAL);
  });
  if (d.M <= 0) return 0;
  k_blocks<P, KIND><<<(unsigned)d.M, TH, L::BYTES_LOCAL, st>>>(d.C, d.mesh, q, qtr, fvn, shift, eps, BT, out_slot);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_coupling(const DiscDev& d, const double* q, const double* qtr, const double* fvn, double eps,
                        int64_t npairs, const int* pair_e, const signed char* pair_f, const int* pair_slot,
                        const signed char* pair_add, double* blocks, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int TH = BC<P>::THREADS;
  static std::atomic<unsigned long long> attr_seen{0};
  once_per_device(attr_seen, [&] {
    cudaFuncSetAttribute(k_coupling<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)L::BYTES_COUPLING);
  });
  if (npairs <= 0) return 0;
  k_coupling<P, KIND><<<(unsigned)npairs, TH, L::BYTES_COUPLING, st>>>(d.C, d.mesh, q, qtr, fvn, eps, pair_e,
                                                                         pair_f, pair_slot, pair_add, blocks);
  return (int)cudaGetLastError();
}

template <int P, int KIND>
static int run_forces(const DiscDev& d, const double* q, int64_t nwall, const int* wall_e,
                      const signed char* wall_f, const double* weights, double* out, cudaStream_t st) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB, TH = BC<P>::THREADS;
  if constexpr (!KT<KIND>::FLOW) {
    return -5;
  } else {
    static std::atomic<unsigned long long> attr_seen{0};
    once_per_device(attr_seen, [&] {
      cudaFuncSetAttribute(k_trace<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_TRACE);
      cudaFuncSetAttribute(k_fvn<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES_FVN);
    });
    const unsigned grid = (unsigned)((d.M + E - 1) / E);
    const unsigned gl = (unsigned)((d.M * 2 * (P + 1) + 127) / 128);
    k_trace_lines<P, KIND><<<gl, 128, 0, st>>>(d.C, d.mesh, q, nullptr, 0.0, nullptr, d.qtr, nullptr);
    if constexpr (KT<KIND>::VISC)
      k_fvn<P, KIND><<<grid, TH, L::BYTES_FVN, st>>>(d.C, d.mesh, q, d.qtr, d.fvn, d.grad, 0);
    FaceWeights fw{};
    for (int k = 0; k <= P; ++k) fw.w[k] = weights[k];
    if (nwall > 0)
      k_wall_forces<P, KIND><<<(unsigned)((nwall + 127) / 128), 128, 0, st>>>(d.C, d.mesh, d.qtr, d.grad, wall_e,
                                                                               wall_f, nwall, fw, out);
    return (int)cudaGetLastError();
  }
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

template <int P, int KIND>
static size_t grad_scratch_doubles_t(int64_t M) {
  using L = SL<P, KIND>;
  constexpr int E = BC<P>::EPB;
  return (size_t)((M + E - 1) / E) * 2 * KT<KIND>::NW * L::PS;
}

size_t fr_grad_scratch_doubles(int p, int kind, int64_t M) {
  switch (kind * 8 + p) {
#define PMGB_GS(K, PP) case K * 8 + PP: return grad_scratch_doubles_t<PP, K>(M);
    PMGB_GS(K_EULER, 0) PMGB_GS(K_EULER, 1) PMGB_GS(K_EULER, 2) PMGB_GS(K_EULER, 3) PMGB_GS(K_EULER, 4) PMGB_GS(K_EULER, 5)
    PMGB_GS(K_NS, 0) PMGB_GS(K_NS, 1) PMGB_GS(K_NS, 2) PMGB_GS(K_NS, 3) PMGB_GS(K_NS, 4) PMGB_GS(K_NS, 5)
    PMGB_GS(K_ADV, 0) PMGB_GS(K_ADV, 1) PMGB_GS(K_ADV, 2) PMGB_GS(K_ADV, 3) PMGB_GS(K_ADV, 4) PMGB_GS(K_ADV, 5)
    PMGB_GS(K_ADVD, 0) PMGB_GS(K_ADVD, 1) PMGB_GS(K_ADVD, 2) PMGB_GS(K_ADVD, 3) PMGB_GS(K_ADVD, 4) PMGB_GS(K_ADVD, 5)
#undef PMGB_GS
  }
  return 0;
}

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
                  double eps, double* BT, cudaStream_t st, const int* out_slot) {
  PMGB_DISPATCH(run_blocks, d, q, qtr, fvn, shift, eps, BT, out_slot, st)
}

int launch_forces(const DiscDev& d, const double* q, int64_t nwall, const int* wall_e, const signed char* wall_f,
                  const double* weights, double* out, cudaStream_t st) {
  PMGB_DISPATCH(run_forces, d, q, nwall, wall_e, wall_f, weights, out, st)
}

int launch_coupling(const DiscDev& d, const double* q, const double* qtr, const double* fvn, double eps,
                    int64_t npairs, const int* pair_e, const signed char* pair_f, const int* pair_slot,
                    const signed char* pair_add, double* blocks, cudaStream_t st) {
  PMGB_DISPATCH(run_coupling, d, q, qtr, fvn, eps, npairs, pair_e, pair_f, pair_slot, pair_add, blocks, st)
}

int* bad_ptr() {
  int* p = nullptr;
  cudaGetSymbolAddress((void**)&p, g_bad);
  return p;
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
