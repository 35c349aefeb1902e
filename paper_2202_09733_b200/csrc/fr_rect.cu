// FR residual R(u) and its fused epilogues on meshes of axis-aligned
// rectangles (every BASELINE.json mesh: periodic boxes and the stretched
// channel) -- hand-written FP64 kernels for sm_100a.
//
// Reference: /root/reference/pkg/src/pmgflow/spatial.py:501-570 (residual),
// 594-603 (BR1 gradients), 407-430 (FR divergence), 113-203 (fluxes).
//
// On a rectangle the bilinear map is x = x0 + a0 xi, y = y0 + d0 eta with
// exactly axis-aligned unit normals and face_jac = a0 (faces 0, 2) and d0
// (faces 1, 3), so the reference's metric terms reduce to per-element
// constants and every cross term is an exact zero:
//   gx = (1/a0) [D_xi W + lR (What_1 - tr_1 W) - lL (What_3 - tr_3 W)]
//   gy = (1/d0) [D_eta W + lR (What_2 - tr_2 W) - lL (What_0 - tr_0 W)]
//   R  = -[(1/a0) X_xi + (1/d0) X_eta],
//   X_xi  = D_xi fx + lR (Fc_1 - tr_1 fx) - lL (-Fc_3 - tr_3 fx)
//   X_eta = D_eta fy + lR (Fc_2 - tr_2 fy) - lL (-Fc_0 - tr_0 fy)
// (the reference's expressions with J = diag(a0, d0) substituted; they
// differ from it only in rounding).  The one-sided viscous normal flux on a
// face is +-fx or +-fy, so only that row of the stress is formed.
//
// Two kernels chained with programmatic dependent launch (navier-stokes;
// for euler the first one is the per-face k_rface).  Both take one thread
// per (element, line); a CTA's contiguous q / What blocks arrive by TMA bulk
// copies (UBLKCP) completed on an mbarrier; the only gathers are the
// neighbours' q lines (k_rgf) and the four face records of a thread
// (k_rasm):
//   k_rgf    traces on the four faces (own: from the staged q block;
//            neighbours: gathered from q), the BR1
//            common value What into the element's own What block, the
//            interface flux F (Roe / Rusanov) once per face by its L side,
//            BR1 gradients by line passes (rows gx, columns gy, one
//            shared-memory transpose each), their face traces, and the
//            element's share of the common total normal flux (spatial.py:
//            559-568) into the face record: G = F - fl/2 from the L side,
//            H = fr/2 from the R side (LDG: G = F, H = fr; boundary: F - fl)
//   k_rasm   Fc = +-(G + H) from the gathered records, gradients again
//            (cheaper than a 2 x 79 MB round trip at config 2), point
//            fluxes, the FR divergence by line passes, the fused epilogue;
//            element blocks in descending order (k_rgf's last blocks are
//            still in L2), epilogue operands prefetched to L2 at the start
// Kept for A/B and as a cross-check (Discretization.residual_path): the
// four-kernel chain this replaced (k_rface + k_rgrad + k_rfc + k_rasm with
// per-element Fc blocks).
// Line threads keep each line in registers, so the operator contractions
// read shared memory only for the transposes (blocks of one line, stride
// an odd number of 16-byte units: conflict-free 128-bit accesses).
#include <climits>

#include "fr_device.cuh"

namespace pmgb {

struct RectMesh {
  int64_t M;
  int64_t nface;
  const int4* __restrict__ faces;    // {eL, fL | rev<<2 | bnd<<3 | tag<<4, eR, fR}
  const int* __restrict__ fslot;     // (M,4) face index of every element face
  const int2* __restrict__ link;     // (M,4) the general link table
  const double2* __restrict__ rgeo;  // (M) {1/a0, 1/d0}
  const double* __restrict__ geom;   // (M,20) for the face normals
};

// Line-block transpose layouts: value pos of line `line` of element el at
// el * S + line * BS + pos.  Row threads write column blocks (scattered
// 64-bit stores), column threads read their own block (64-bit loads); S and
// BS are the smallest strides that keep both patterns at the minimum
// number of shared-memory wavefronts per warp (or close to it), from an
// exhaustive search over the thread -> (element, line) map of the CTA
// (tools/bank_model.py): V = 3 values per line point (W, gx, gy), V = 4
// (fy, X_xi).
template <int N, int V> struct TL;
template <> struct TL<2, 3> { static constexpr int BS = 7, S = 14; };
template <> struct TL<2, 4> { static constexpr int BS = 9, S = 18; };
template <> struct TL<3, 3> { static constexpr int BS = 17, S = 51; };
template <> struct TL<3, 4> { static constexpr int BS = 17, S = 51; };
template <> struct TL<4, 3> { static constexpr int BS = 13, S = 52; };
template <> struct TL<4, 4> { static constexpr int BS = 17, S = 68; };
template <> struct TL<5, 3> { static constexpr int BS = 17, S = 85; };
template <> struct TL<5, 4> { static constexpr int BS = 20, S = 101; };
template <> struct TL<6, 3> { static constexpr int BS = 21, S = 126; };
template <> struct TL<6, 4> { static constexpr int BS = 25, S = 150; };
template <int N, int V>
__host__ __device__ constexpr int tl(int el, int line, int pos) {
  return el * TL<N, V>::S + line * TL<N, V>::BS + pos;
}

// per-face-point record of the unique-face array: F on L's normal, then the
// one-sided viscous fluxes of the L and R sides on their own normals
constexpr int FREC4 = 12;
// Two-kernel chain.  PMGB_RECT_REC12 = 1 (default): the same 12-double
// record [F | fl | fr], the L side writing F and fl, the R side fr, and
// k_rasm forming Fc = F - 0.5 (fl - fr) as the reference rounds it
// (spatial.py:559-568; k_rfc's arithmetic).
// PMGB_RECT_REC12 = 0: 8 doubles, [0..3] G = F - (L's share of the common
// viscous flux) from the L side, [4..6] H = the R side's share, Fc = G + H:
// a third less record traffic (config-2 R 114.6 -> 105.0 us,
// profiles/r2/ab_rec12_r2t.log), but (F - fl/2) + fr/2 rounds F's
// magnitude once more than the reference does; through the FD products
// that moved one restarted-GMRES count of the 48^2 config-2 step from
// within 1 to within 2 of the reference's (tests/test_gpu_fullsize_oracle.py),
// so it is not the default.
#ifndef PMGB_RECT_REC12
#define PMGB_RECT_REC12 1
#endif
constexpr int FREC = PMGB_RECT_REC12 ? 12 : 8;

// CTA width target of the element kernels: 64 threads (12 elements at p = 4,
// six CTAs per SM) interleave the CTAs' load and compute phases more finely than
// 128 (config-2 R 105.9 -> 105.1 us, config 4 87.3 -> 85.9; 96: 108.6 / 86.0, 48: 117.2 / 91.5;
// profiles/r2/ab_xch_r2n.log, ab_cta_width_r2t.log)
#ifndef PMGB_RECT_TH
#define PMGB_RECT_TH 64
#endif
// k_rgf: a neighbour that sits in the CTA's own staged q block is read from
// shared memory instead of being gathered from global memory (same operands,
// same order: bitwise the gathered trace)
// -1: per degree (RC<P>::NBS); 0 off, 1 in the Jv forms only, 2 always
#ifndef PMGB_RECT_NBS
#define PMGB_RECT_NBS -1
#endif
// k_rgf / k_rasm: rows of the staged q (and X) block padded by this many
// doubles (one bulk copy per row): at the raw row stride of N * 32 B the line
// threads' 128-bit row reads collide in the banks (2-way at p = 4, 8-way at
// p = 3, 4-way at p = 5); + 16 B makes every quarter-warp conflict-free
// -1: per degree (RC<P>::QPAD)
#ifndef PMGB_RECT_QPAD
#define PMGB_RECT_QPAD -1
#endif
// NS two-kernel chain: the 12-double records of a face laid out part by part
// ([F of the N points | fl | fr]) instead of point by point, so the line
// threads of an element touch 2 cache lines per 256-bit record access, not 4
// (config-2 R 105.0 -> 102.8 us, Jv 142.8 -> 139.1; config 4 R 74.1 -> 71.9;
// bitwise the same results; profiles/r2/ab_rsoa_r2y.log)
#ifndef PMGB_RECT_RSOA
#define PMGB_RECT_RSOA 1
#endif
// k_rgf: the CTA's What block staged in shared memory and written by one bulk
// store instead of 12 scattered 8-byte stores per thread.  -1: where it
// measured faster (p = 4, R / defect forms: config-2 R 102.7 -> 101.3 us; the
// Jv forms and p = 3 lose 0.5-1.5 %; profiles/r2/ab_wtma_r2y.log), 0 off, 1 on
#ifndef PMGB_RECT_WTMA
#define PMGB_RECT_WTMA -1
#endif
#ifndef PMGB_RECT_PF   // L2 prefetch distance in CTAs (0: off; 888 and 1776 measured slower, ab_cta_width_r2t.log)
#define PMGB_RECT_PF 0
#endif
// k_rasm (two-kernel chain) walks the element blocks in descending order: what
// k_rgf touched last is still in L2 (config-2 R 110.7 -> 105.0 us, Jv 159.2 ->
// 152.2 us; profiles/r2/ab_rev_r2q.log)
#ifndef PMGB_RECT_REV
#define PMGB_RECT_REV 1
#endif
template <int P> struct RC {
  static constexpr int N = P + 1, NP = N * N;
  static constexpr int EPB = PMGB_RECT_TH / N;  // elements per CTA
  static constexpr int TH = EPB * N;   // one thread per (element, line)
  // line block strides in doubles: >= 3N (gradient passes) / 4N (flux
  // passes), even, an odd number of 16-byte units

  // measured per degree (profiles/r2/ab_qpad_nbs_r2y.log): one bulk copy per
  // row costs more than the 2-way conflicts it removes at p = 4
  static constexpr int QPAD = PMGB_RECT_QPAD >= 0 ? PMGB_RECT_QPAD : (P == 3 ? 2 : 0);
  static constexpr int NBS = PMGB_RECT_NBS >= 0 ? PMGB_RECT_NBS : (P == 3 ? 2 : (P >= 4 ? 1 : 0));
  static constexpr int RS = N * 4 + QPAD;  // row stride of a staged q block (k_rgf / k_rasm)
  static constexpr int QD = EPB * N * RS;   // doubles of a q block
  static constexpr int WD = EPB * 4 * N * 3;  // of a What block
  static constexpr int FD = EPB * 4 * N * 4;  // of an Fc block
  // CTAs per SM the register target is set for
#ifdef PMGB_RECT_MINB   // experiment builds: resident CTAs per SM at every degree
  static constexpr int MINB = PMGB_RECT_MINB;
#else
  static constexpr int MINB = (P == 5 ? 2 : (P >= 3 ? 3 : 4)) * (128 / PMGB_RECT_TH);
#endif
};

// q (+ eps X with the reference's rounding, newton_krylov.py:76) of point pt
template <bool HASX>
__device__ __forceinline__ void ld_q(const double* __restrict__ q, const double* __restrict__ X, double eps,
                                     int64_t pt, double* o) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
               : "l"(q + pt * 4));
  if constexpr (HASX) {
    double x[4];
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                 : "l"(X + pt * 4));
#pragma unroll
    for (int v = 0; v < 4; ++v) o[v] = __dadd_rn(o[v], __dmul_rn(eps, x[v]));
  }
}

// primitive variables of one state, exactly as prim() (spatial.py:94-101)
struct Pr {
  double r, ir, u, v, p;
};
__device__ __forceinline__ Pr prim_of(const double* q, double g) {
  Pr s;
  prim(q, g, s.r, s.ir, s.u, s.v, s.p);
  return s;
}

// Roe flux from precomputed primitives: the same expressions as roe()
// (spatial.py:113-163), so the result is bitwise roe(qL, qR, ...)
__device__ __forceinline__ void roe_pr(const double* qL, const Pr& L, const double* qR, const Pr& R, double nx,
                                       double ny, double g, double* F) {
  const double EpL = qL[3] + L.p, EpR = qR[3] + R.p;
  const double HL = EpL * L.ir;
  const double HR = EpR * R.ir;
  const double sL = fsqrt(L.r), sR = fsqrt(R.r);
  const double w = sL * rcp(sL + sR), w1 = 1.0 - w;
  const double u = w * L.u + w1 * R.u;
  const double v = w * L.v + w1 * R.v;
  const double H = w * HL + w1 * HR;
  const double ke = 0.5 * (u * u + v * v);
  const double c2 = (g - 1.0) * (H - ke);
  const double c = fsqrt(c2);
  const double ic2 = rcp(c2);
  const double rb = sL * sR;
  const double un = u * nx + v * ny;
  const double du = R.u - L.u, dv = R.v - L.v;
  const double dn = du * nx + dv * ny;
  const double dtg = -du * ny + dv * nx;
  const double dp = R.p - L.p;
  const double k1 = fabs(un - c) * ((dp - rb * c * dn) * (0.5 * ic2));
  const double k2 = fabs(un) * ((R.r - L.r) - dp * ic2);
  const double k3 = fabs(un) * (rb * dtg);
  const double k4 = fabs(un + c) * ((dp + rb * c * dn) * (0.5 * ic2));
  const double ut = -u * ny + v * nx;
  const double d0 = k1 + k2 + k4;
  const double d1 = k1 * (u - c * nx) + k2 * u - k3 * ny + k4 * (u + c * nx);
  const double d2 = k1 * (v - c * ny) + k2 * v + k3 * nx + k4 * (v + c * ny);
  const double d3 = k1 * (H - c * un) + k2 * ke + k3 * ut + k4 * (H + c * un);
  const double qnL = L.u * nx + L.v * ny, qnR = R.u * nx + R.v * ny;
  F[0] = 0.5 * (qL[0] * qnL + qR[0] * qnR) - 0.5 * d0;
  F[1] = 0.5 * ((qL[1] * qnL + L.p * nx) + (qR[1] * qnR + R.p * nx)) - 0.5 * d1;
  F[2] = 0.5 * ((qL[2] * qnL + L.p * ny) + (qR[2] * qnR + R.p * ny)) - 0.5 * d2;
  F[3] = 0.5 * (EpL * qnL + EpR * qnR) - 0.5 * d3;
}

// Rusanov from primitives: the same expressions as rusanov()
__device__ __forceinline__ void rusanov_pr(const double* qL, const Pr& L, const double* qR, const Pr& R, double nx,
                                           double ny, double g, double* F) {
  const double qnL = L.u * nx + L.v * ny, qnR = R.u * nx + R.v * ny;
  const double lam = fmax(fabs(qnL) + fsqrt(g * L.p * L.ir), fabs(qnR) + fsqrt(g * R.p * R.ir));
  const double hl = 0.5 * lam;
  F[0] = 0.5 * (qL[0] * qnL + qR[0] * qnR) - hl * (qR[0] - qL[0]);
  F[1] = 0.5 * ((qL[1] * qnL + L.p * nx) + (qR[1] * qnR + R.p * nx)) - hl * (qR[1] - qL[1]);
  F[2] = 0.5 * ((qL[2] * qnL + L.p * ny) + (qR[2] * qnR + R.p * ny)) - hl * (qR[2] - qL[2]);
  F[3] = 0.5 * ((qL[3] + L.p) * qnL + (qR[3] + R.p) * qnR) - hl * (qR[3] - qL[3]);
}

// trace of q (+ eps X) on face f at face point k: line sum over the line
// through that point in line_sum's order (i = 0..N-1 along the line)
// chk: also report whether every point of the line is physical (Euler
// kinds, which have no k_rgrad to check the states)
template <int P, bool HASX>
__device__ __forceinline__ void face_trace(const FrConst& C, const double* __restrict__ q,
                                           const double* __restrict__ X, double eps, int64_t e, int f, int k,
                                           double* tr, bool chk = false, bool* ok = nullptr) {
  constexpr int N = P + 1, NP = N * N;
  const bool col = (f == 0 || f == 2);
  const int kk = (f >= 2) ? N - 1 - k : k;   // the row / column index
  const int start = col ? kk : kk * N;
  const int step = col ? N : 1;
  const double* w = (f == 1 || f == 2) ? C.eR : C.eL;
  tr[0] = tr[1] = tr[2] = tr[3] = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x[4];
    ld_q<HASX>(q, X, eps, e * NP + start + i * step, x);
    if (chk) *ok = *ok && physical(x, C.gamma);
    const double wi = w[i];
#pragma unroll
    for (int v = 0; v < 4; ++v) tr[v] += wi * x[v];
  }
}

// ---------------------------------------------------------------------------
// 256-bit global accesses (LDG/STG.E.ENL2.256 on sm_100a)

__device__ __forceinline__ void ldg4(const double* __restrict__ p, double* o) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
}
// coherent (L1-bypassing is not needed: written by an earlier kernel)
__device__ __forceinline__ void ldg4c(const double* p, double* o) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
}
__device__ __forceinline__ void stg4(double* p, const double* v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}

// The epilogue operands of one point (4 variables) as 256-bit loads:
// epi_load_k's operands (fr_device.cuh), o*[v] for variable v
template <int EK>
__device__ __forceinline__ void epi_load4_k(const Epi& ep, int64_t i, double* o1, double* o2, double* o3) {
  if constexpr (EK < 0) {
#pragma unroll
    for (int v = 0; v < 4; ++v) epi_load_k<EK>(ep, i + v, o1[v], o2[v], o3[v]);
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v) o1[v] = o2[v] = o3[v] = 0.0;
    constexpr bool SBSE = EK == EPI_DEFECT || EK == EPI_RK;
    if constexpr (EK == EPI_JV || EK == EPI_STAGE_JV) {
      ldg4(ep.X + i, o1);
      ldg4(ep.R0 + i, o2);
    }
    if constexpr (EK == EPI_STAGE_F || EK == EPI_STAGE_JV) ldg4(ep.E + i, o3);
    if constexpr (SBSE) {
      if (ep.Sb)
        ldg4(ep.Sb + i, o1);
      else
        o1[0] = o1[1] = o1[2] = o1[3] = ep.sb_scalar;
    }
    if constexpr (SBSE || EK == EPI_OUTER_F) {
      if (ep.Se)
        ldg4(ep.Se + i, o2);
      else
        o2[0] = o2[1] = o2[2] = o2[3] = ep.se_scalar;
    }
    if constexpr (EK == EPI_RK) ldg4(ep.Q0 + i, o3);
  }
}

// L2 prefetch of the epilogue operands of a CTA's element block (issued at
// kernel start: the operands are inputs of the whole chain), so that the
// loads at the end of the kernel find them in L2
// epilogue operand request distance in points (0: at the point itself); measured
// (profiles/r2/ab_epd_r2x.log): 1 takes 1-2 % off the Jv / stage-Jv / defect forms
#ifndef PMGB_RECT_EPD
#define PMGB_RECT_EPD 1
#endif
#ifndef PMGB_RECT_EPF   // measured: config-2 Jv 166.4 -> 161.3 us (profiles/r2/ab_pdl0_epf_r2p.log)
#define PMGB_RECT_EPF 1
#endif
__device__ __forceinline__ void l2_prefetch_blk(const double* p, int64_t off, uint32_t bytes) {
  if (p != nullptr)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(bytes) : "memory");
}
template <int EK>
__device__ __forceinline__ void epi_prefetch(const Epi& ep, int64_t off, uint32_t bytes) {
  if constexpr (EK == EPI_JV || EK == EPI_STAGE_JV) {
    l2_prefetch_blk(ep.X, off, bytes);
    l2_prefetch_blk(ep.R0, off, bytes);
  }
  if constexpr (EK == EPI_STAGE_F || EK == EPI_STAGE_JV) l2_prefetch_blk(ep.E, off, bytes);
  if constexpr (EK == EPI_DEFECT || EK == EPI_RK) l2_prefetch_blk(ep.Sb, off, bytes);
  if constexpr (EK == EPI_DEFECT || EK == EPI_RK || EK == EPI_OUTER_F) l2_prefetch_blk(ep.Se, off, bytes);
  if constexpr (EK == EPI_RK) l2_prefetch_blk(ep.Q0, off, bytes);
}

// L2 residency hints across the chain (126 MB L2; working set ~190 MB at
// config 2): intermediates stored evict_last, inputs loaded evict_first on
// their last read of the chain (k_rasm).  Measured slower (config-2 R
// 117.1 -> 120.6 us, profiles/r2/ab_l2_hints_r2.log): off by default.
#ifndef PMGB_RECT_L2_HINTS
#define PMGB_RECT_L2_HINTS 0
#endif
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void stg4_last(double* p, const double* v) {
#if PMGB_RECT_L2_HINTS
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v[0]), "d"(v[1]),
               "d"(v[2]), "d"(v[3]), "l"(pol_last())
               : "memory");
#else
  stg4(p, v);
#endif
}
// the chain's output: nothing in the chain reads it again
__device__ __forceinline__ void stg4_first(double* p, const double* v) {
#if PMGB_RECT_L2_HINTS
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v[0]), "d"(v[1]),
               "d"(v[2]), "d"(v[3]), "l"(pol_first())
               : "memory");
#else
  stg4(p, v);
#endif
}
__device__ __forceinline__ void stg1_last(double* p, double v) {
#if PMGB_RECT_L2_HINTS
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol_last()) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void ldg4_first(const double* p, double* o) {
#if PMGB_RECT_L2_HINTS
  asm volatile("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]),
               "=d"(o[3]) : "l"(p), "l"(pol_first()));
#else
  ldg4c(p, o);
#endif
}

// ---------------------------------------------------------------------------
// k_rface: traces, interface flux and BR1 common value, once per face point

template <int P, int KIND, bool HASX, int RS = FREC4>
__global__ void __launch_bounds__(128) k_rface(const FrConst C, const RectMesh m, const double* __restrict__ q,
                                               const double* __restrict__ X, double eps, double* __restrict__ frec,
                                               double* __restrict__ wh, int* __restrict__ bad) {
  constexpr int N = P + 1;
  constexpr bool VISC = KT<KIND>::VISC;
  const int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (t >= m.nface * N) return;
  const int64_t phi = t / N;
  const int k = (int)(t - phi * N);
  const int4 fr = __ldg(m.faces + phi);
  const int fL = fr.y & 3, rev = (fr.y >> 2) & 1, bnd = (fr.y >> 3) & 1, tag = (fr.y >> 4) & 15;
  const double2 nrm = __ldg(reinterpret_cast<const double2*>(m.geom + (int64_t)fr.x * 20 + 8 + 2 * fL));
  const double g = C.gamma;
  const Phys ph = phys_of(C);
  const int kk = rev ? N - 1 - k : k;
  // the stream predecessor (launched ahead of with programmatic
  // serialization) may still be writing q or reading the records
  pdl_wait();
  pdl_trigger();
  double qa[4], qc[4];
  // Euler: the states are checked here, on the rows of each element's face 1
  bool okL = true, okR = true;
  const bool chk = !VISC && bad != nullptr;
  face_trace<P, HASX>(C, q, X, eps, fr.x, fL, k, qa, chk && fL == 1, &okL);
  if (bnd)
    ghost<KIND>(qa, tag, nrm.x, nrm.y, C.qinf, qc);
  else
    face_trace<P, HASX>(C, q, X, eps, fr.z, fr.w, kk, qc, chk && fr.w == 1, &okR);
  if (!okL) atomicMin(bad, fr.x);
  if (!okR) atomicMin(bad, fr.z);
  const Pr A = prim_of(qa, g), B = prim_of(qc, g);
  if (bad != nullptr) {
    if (!(A.r > 0.0 && A.p > 0.0)) atomicMin(bad + 1, fr.x);
    if (!bnd && !(B.r > 0.0 && B.p > 0.0)) atomicMin(bad + 1, fr.z);
  }
  double F[4];
  if (ph.riemann)
    rusanov_pr(qa, A, qc, B, nrm.x, nrm.y, g, F);
  else
    roe_pr(qa, A, qc, B, nrm.x, nrm.y, g, F);
  stg4_last(frec + t * RS, F);
  if constexpr (VISC) {
    double wa[3] = {A.u, A.v, A.p * A.ir}, wc[3] = {B.u, B.v, B.p * B.ir};
    if (bnd) ghost_w<KIND>(ph, tag, wa, wc);
    double w[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = common_w(ph, !bnd, true, wa[c], wc[c]);
    double* dL = wh + (((int64_t)fr.x * 4 + fL) * N + k) * 3;
    stg1_last(dL, w[0]), stg1_last(dL + 1, w[1]), stg1_last(dL + 2, w[2]);
    if (!bnd) {
      double* dR = wh + (((int64_t)fr.z * 4 + fr.w) * N + kk) * 3;
      stg1_last(dR, w[0]), stg1_last(dR + 1, w[1]), stg1_last(dR + 2, w[2]);
    }
  }
}

// ---------------------------------------------------------------------------
// k_rfc: the common total normal flux, once per face point, to both sides

template <int P, int KIND>
__global__ void __launch_bounds__(128) k_rfc(const FrConst C, const RectMesh m, const double* __restrict__ frec,
                                             double* __restrict__ fc) {
  constexpr int N = P + 1;
  pdl_trigger();
  const int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const bool live = t < m.nface * N;
  const int64_t phi = live ? t / N : 0;
  const int k = (int)(t - phi * N);
  const int4 fr = live ? __ldg(m.faces + phi) : make_int4(0, 0, 0, 0);
  pdl_wait();  // frec (k_rface F, k_rgrad fvn)
  if (!live) return;
  const int fL = fr.y & 3, rev = (fr.y >> 2) & 1, bnd = (fr.y >> 3) & 1, tag = (fr.y >> 4) & 15;
  const Phys ph = phys_of(C);
  const double* rec = frec + t * FREC4;
  double Fc[4];
  ldg4_first(rec, Fc);
  if constexpr (KT<KIND>::VISC) {
    double fl[4], fr_[4], Fv[4];
    ldg4_first(rec + 4, fl);
    if (bnd) {
#pragma unroll
      for (int v = 0; v < 4; ++v) Fv[v] = common_fv(ph, false, true, fl[v], fl[v]);
      if (tag == T_WALL_ADIABATIC) Fv[3] = 0.0;
    } else {
      ldg4_first(rec + 8, fr_);
#pragma unroll
      for (int v = 0; v < 4; ++v) Fv[v] = common_fv(ph, true, true, fl[v], fr_[v]);
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) Fc[v] = Fc[v] - Fv[v];
  }
  stg4_last(fc + (((int64_t)fr.x * 4 + fL) * N + k) * 4, Fc);
  if (!bnd) {
    const double n[4] = {-Fc[0], -Fc[1], -Fc[2], -Fc[3]};
    stg4_last(fc + (((int64_t)fr.z * 4 + fr.w) * N + (rev ? N - 1 - k : k)) * 4, n);
  }
}

// ---------------------------------------------------------------------------
// shared by the element kernels

// TMA bulk copy of a contiguous global block into shared memory, completed
// on an mbarrier (UBLKCP + SYNCS)
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
// the same with an L2 evict_first policy (the block's last read in the chain)
__device__ __forceinline__ void bulk_g2s_first(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
#if PMGB_RECT_L2_HINTS
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar)), "l"(pol_first())
      : "memory");
#else
  bulk_g2s(dst, src, bytes, bar);
#endif
}
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n RW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra RW%=;\n}" ::"r"(
          saddr(bar)),
      "r"(phase)
      : "memory");
}

// q + eps X formed in place in the staged q block (the reference's rounding)
template <int TH>
__device__ __forceinline__ void form_qp(double* sQ, const double* sXb, double eps, int nd) {
  for (int i = 2 * threadIdx.x; i < nd; i += 2 * TH) {
    double2 a = *reinterpret_cast<const double2*>(sQ + i);
    const double2 x = *reinterpret_cast<const double2*>(sXb + i);
    a.x = __dadd_rn(a.x, __dmul_rn(eps, x.x));
    a.y = __dadd_rn(a.y, __dmul_rn(eps, x.y));
    *reinterpret_cast<double2*>(sQ + i) = a;
  }
}

// one point of a staged q block
__device__ __forceinline__ void lds4(const double* p, double* o) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  o[0] = a.x;
  o[1] = a.y;
  o[2] = b.x;
  o[3] = b.y;
}

// the CTA's q (+ X) rows into the (padded) staged block: one bulk copy for the
// block, or one per row by its line thread when the rows are padded
template <int P, bool HASX, bool FIRST>
__device__ __forceinline__ void stage_q(double* sQ, double* sX, const double* __restrict__ q,
                                        const double* __restrict__ X, int64_t e0, int ne, uint64_t* bar) {
  using R = RC<P>;
  constexpr int N = R::N, NP = R::NP;
  const int t = threadIdx.x;
  const uint32_t qbytes = (uint32_t)ne * NP * 32;
  if (t == 0) mbar_expect(bar, HASX ? 2 * qbytes : qbytes);
  if constexpr (R::QPAD > 0) {
    if (t < ne * N) {
      const double* src = q + (e0 * NP + (int64_t)t * N) * 4;
      if (FIRST) bulk_g2s_first(sQ + t * R::RS, src, N * 32, bar);
      else bulk_g2s(sQ + t * R::RS, src, N * 32, bar);
      if (HASX) bulk_g2s(sX + t * R::RS, X + (e0 * NP + (int64_t)t * N) * 4, N * 32, bar);
    }
  } else if (t == 0) {
    if (FIRST) bulk_g2s_first(sQ, q + e0 * NP * 4, qbytes, bar);
    else bulk_g2s(sQ, q + e0 * NP * 4, qbytes, bar);
    if (HASX) bulk_g2s(sX, X + e0 * NP * 4, qbytes, bar);
  }
}
// q + eps X in place, row by row (the rows may be padded)
template <int P>
__device__ __forceinline__ void form_qp_rows(double* sQ, const double* sXb, double eps, int ne) {
  using R = RC<P>;
  if constexpr (R::QPAD > 0) {
    const int t = threadIdx.x;
    if (t < ne * R::N) {
#pragma unroll
      for (int i = 0; i < R::N * 4; i += 2) {
        double2 a = *reinterpret_cast<const double2*>(sQ + t * R::RS + i);
        const double2 x = *reinterpret_cast<const double2*>(sXb + t * R::RS + i);
        a.x = __dadd_rn(a.x, __dmul_rn(eps, x.x));
        a.y = __dadd_rn(a.y, __dmul_rn(eps, x.y));
        *reinterpret_cast<double2*>(sQ + t * R::RS + i) = a;
      }
    }
  } else {
    form_qp<R::TH>(sQ, sXb, eps, ne * R::NP * 4);
  }
}

// face_trace() on a staged q block (q + eps X already formed in place)
template <int P>
__device__ __forceinline__ void face_trace_s(const FrConst& C, const double* sQ, int el, int f, int k, double* tr) {
  constexpr int N = P + 1, NP = N * N;
  const bool col = (f == 0 || f == 2);
  const int kk = (f >= 2) ? N - 1 - k : k;
  const int start = col ? kk : kk * N;
  const int step = col ? N : 1;
  const double* w = (f == 1 || f == 2) ? C.eR : C.eL;
  tr[0] = tr[1] = tr[2] = tr[3] = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x[4];
    const int pt = start + i * step;
    lds4(sQ + (el * N + pt / N) * RC<P>::RS + (pt % N) * 4, x);
    const double wi = w[i];
#pragma unroll
    for (int v = 0; v < 4; ++v) tr[v] += wi * x[v];
  }
}

// face points of line thread a: [0] face 0 point a, [1] face 1 point a,
// [2] face 2 point N-1-a, [3] face 3 point N-1-a
template <int N>
__device__ __forceinline__ int fpt_of(int f, int a) {
  return f * N + ((f >= 2) ? N - 1 - a : a);
}

// BR1 gradient along one line (row: gx with ia; column: gy with id) from
// the line's viscous variables w[c][i] and the common values at its two
// ends: wp on the +1 end (eR, lR), wm on the -1 end (eL, lL)
template <int N>
__device__ __forceinline__ void line_gradient(const FrConst& C, const double (&w)[3][N], const double* wp,
                                              const double* wm, double s, double (&gr)[3][N]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double tp = 0.0, tm = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      tp += C.eR[i] * w[c][i];
      tm += C.eL[i] * w[c][i];
    }
    const double cp = wp[c] - tp, cm = wm[c] - tm;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double d = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) d += C.D[b * N + i] * w[c][i];
      gr[c][b] = s * ((d + C.lR[b] * cp) - C.lL[b] * cm);
    }
  }
}

// x-row (fx) / y-row (fy) of the viscous flux at one state, exactly the
// corresponding components of visc_flux() (spatial.py:166-180)
__device__ __forceinline__ void visc_fx(const double* q, const double* gx, const double* gy, const Phys& ph,
                                        double* fx) {
  const double ir = rcp(q[0]);
  const double u = q[1] * ir, v = q[2] * ir;
  const double d = gx[0] + gy[1];
  const double txx = ph.mu * (2.0 * gx[0] - (2.0 / 3.0) * d);
  const double txy = ph.mu * (gy[0] + gx[1]);
  fx[0] = 0.0;
  fx[1] = txx;
  fx[2] = txy;
  fx[3] = u * txx + v * txy + ph.kappa * gx[2];
}
__device__ __forceinline__ void visc_fy(const double* q, const double* gx, const double* gy, const Phys& ph,
                                        double* fy) {
  const double ir = rcp(q[0]);
  const double u = q[1] * ir, v = q[2] * ir;
  const double d = gx[0] + gy[1];
  const double tyy = ph.mu * (2.0 * gy[1] - (2.0 / 3.0) * d);
  const double txy = ph.mu * (gy[0] + gx[1]);
  fy[0] = 0.0;
  fy[1] = txy;
  fy[2] = tyy;
  fy[3] = u * txy + v * tyy + ph.kappa * gy[2];
}

// the same from the trace state's velocity (u, v as prim() forms them)
__device__ __forceinline__ void visc_fx_uv(double u, double v, const double* gx, const double* gy, const Phys& ph,
                                           double* fx) {
  const double d = gx[0] + gy[1];
  const double txx = ph.mu * (2.0 * gx[0] - (2.0 / 3.0) * d);
  const double txy = ph.mu * (gy[0] + gx[1]);
  fx[0] = 0.0;
  fx[1] = txx;
  fx[2] = txy;
  fx[3] = u * txx + v * txy + ph.kappa * gx[2];
}
__device__ __forceinline__ void visc_fy_uv(double u, double v, const double* gx, const double* gy, const Phys& ph,
                                           double* fy) {
  const double d = gx[0] + gy[1];
  const double tyy = ph.mu * (2.0 * gy[1] - (2.0 / 3.0) * d);
  const double txy = ph.mu * (gy[0] + gx[1]);
  fy[0] = 0.0;
  fy[1] = txy;
  fy[2] = tyy;
  fy[3] = u * txy + v * tyy + ph.kappa * gy[2];
}

// divergence along one line of a 4-variable flux x[v][i]: the +1 end takes
// (Fp - trace), the -1 end (-Fm - trace)  (the reference's c1/c3, c2/c0)
template <int N>
__device__ __forceinline__ void line_div(const FrConst& C, const double (&x)[4][N], const double* Fp,
                                         const double* Fm, double (&out)[4][N]) {
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    double tp = 0.0, tm = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      tp += C.eR[i] * x[v][i];
      tm += C.eL[i] * x[v][i];
    }
    const double cp = Fp[v] - tp, cm = -Fm[v] - tm;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double d = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) d += C.D[b * N + i] * x[v][i];
      out[v][b] = (d + C.lR[b] * cp) - C.lL[b] * cm;
    }
  }
}

// ---------------------------------------------------------------------------
// k_rgrad: BR1 gradients, their face traces, one-sided viscous fluxes

// shared memory: [q block | stage]; the stage first holds the X block (Jv
// forms, at its start) and the What block (at its end), then the two
// line-block transposes
template <int P, bool HASX> struct GL {
  using R = RC<P>;
  static constexpr int BUF = R::EPB * TL<R::N, 3>::S;
  static constexpr int A = 2 * BUF, B = R::WD + (HASX ? R::QD : 0);
  static constexpr int STAGE = A > B ? A : B;
  static constexpr int OFF_W = R::QD + STAGE - R::WD, OFF_BAR = R::QD + STAGE;
  static constexpr size_t BYTES = sizeof(double) * (OFF_BAR + 2);
};

template <int P, bool HASX>
__global__ void __launch_bounds__(RC<P>::TH, RC<P>::MINB)
k_rgrad(const FrConst C, const RectMesh m, const double* __restrict__ q, const double* __restrict__ X, double eps,
        const double* __restrict__ wh, double* __restrict__ frec, int* __restrict__ bad) {
  using R = RC<P>;
  using L = GL<P, HASX>;
  constexpr int N = R::N, NP = R::NP, E = R::EPB;
  extern __shared__ __align__(128) double sm[];
  double* sQ = sm;
  double* sX = sm + R::QD;            // X block; then W, then gx (column blocks)
  double* sY = sm + R::QD + L::BUF;   // gy (row blocks)
  const double* sWb = sm + L::OFF_W;  // What block [el][f][k][3]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  const int t = threadIdx.x;
  const int el = t / N, a = t % N;  // row a of element el; also column a
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int ne = (int)((m.M - e0) < E ? (m.M - e0) : E);
  const int64_t e = e0 + el;
  const bool live = t < E * N && el < ne;
  const Phys ph = phys_of(C);
  const double g = C.gamma;
  if (t == 0) {
    mbar_init(bar);
    mbar_init(bar + 1);
  }
  __syncthreads();
  const uint32_t qbytes = (uint32_t)ne * NP * 32;
  if (t == 0) {  // q (+ X): inputs of the chain, before the dependency wait
    mbar_expect(bar, HASX ? 2 * qbytes : qbytes);
    bulk_g2s(sQ, q + e0 * NP * 4, qbytes, bar);
    if (HASX) bulk_g2s(sX, X + e0 * NP * 4, qbytes, bar);
  }
  // static face data of the thread's four face points
  int ri[4] = {0, 0, 0, 0};
  bool lft[4] = {true, true, true, true};
  const double2 rg = live ? __ldg(m.rgeo + e) : make_double2(0.0, 0.0);
  if (live) {
    const int4 sl = __ldg(reinterpret_cast<const int4*>(m.fslot) + e);
    const int4 l01 = __ldg(reinterpret_cast<const int4*>(m.link) + 2 * e);
    const int4 l23 = __ldg(reinterpret_cast<const int4*>(m.link) + 2 * e + 1);
    const int slot[4] = {sl.x, sl.y, sl.z, sl.w};
    const int2 lk[4] = {make_int2(l01.x, l01.y), make_int2(l01.z, l01.w), make_int2(l23.x, l23.y),
                        make_int2(l23.z, l23.w)};
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int k = (f >= 2) ? N - 1 - a : a;
      lft[f] = lk[f].x < 0 || lk_left(lk[f].y);
      const int kL = (!lft[f] && lk_rev(lk[f].y)) ? N - 1 - k : k;
      ri[f] = slot[f] * N + kL;
    }
  }
  pdl_wait();  // What (k_rface)
  if (t == 0) {
    mbar_expect(bar + 1, (uint32_t)ne * 4 * N * 24);
    bulk_g2s(sm + L::OFF_W, wh + e0 * 4 * N * 3, (uint32_t)ne * 4 * N * 24, bar + 1);
  }
  mbar_wait(bar, 0);
  if constexpr (HASX) {
    form_qp<R::TH>(sQ, sX, eps, ne * NP * 4);
    __syncthreads();
  }
  // rows: primitives, W, the row's q traces on faces 1 and 3
  double w[3][N];
  double t1q[4] = {0, 0, 0, 0}, t3q[4] = {0, 0, 0, 0};
  {
    bool ok = true;
    const double* row = sQ + (el * N + a) * N * 4;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double x[4];
      lds4(row + 4 * i, x);
      const Pr s = prim_of(x, g);
      ok = ok && (s.r > 0.0) && (s.p > 0.0);
      w[0][i] = s.u;
      w[1][i] = s.v;
      w[2][i] = s.p * s.ir;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        t1q[v] += C.eR[i] * x[v];
        t3q[v] += C.eL[i] * x[v];
      }
    }
    if (live && !ok && bad != nullptr) atomicMin(bad, (int)e);
  }
  mbar_wait(bar + 1, 0);
  double whv[4][3];
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int c = 0; c < 3; ++c) whv[f][c] = sWb[(el * 4 * N + fpt_of<N>(f, a)) * 3 + c];
  __syncthreads();  // the stage (X, What blocks) is free
  // W into column blocks: block (el, i) holds column i, [c][row]
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) sX[tl<N, 3>(el, i, c * N + a)] = w[c][i];
  // gx along row a (faces 1 and 3)
  double gx[3][N];
  line_gradient<N>(C, w, whv[1], whv[3], rg.x, gx);
  __syncthreads();
  // column a: W of the column, gy (faces 2 and 0)
  double gy[3][N];
  {
    const double* blk = sX + tl<N, 3>(el, a, 0);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int i = 0; i < N; ++i) w[c][i] = blk[c * N + i];
    line_gradient<N>(C, w, whv[2], whv[0], rg.y, gy);
  }
  __syncthreads();  // W reads done
  // gx rows -> column blocks of sX; gy columns -> row blocks of sY
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      sX[tl<N, 3>(el, i, c * N + a)] = gx[c][i];
      sY[tl<N, 3>(el, i, c * N + a)] = gy[c][i];
    }
  // traces of the own-line components: gx on faces 1/3, gy on faces 0/2
  double tgx1[3], tgx3[3], tgy0[3], tgy2[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double s1 = 0.0, s3 = 0.0, s0 = 0.0, s2 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s1 += C.eR[i] * gx[c][i];
      s3 += C.eL[i] * gx[c][i];
      s2 += C.eR[i] * gy[c][i];
      s0 += C.eL[i] * gy[c][i];
    }
    tgx1[c] = s1;
    tgx3[c] = s3;
    tgy2[c] = s2;
    tgy0[c] = s0;
  }
  __syncthreads();
  if (!live) return;
  // rows: gy along row a -> gy traces on faces 1/3; columns: gx -> faces 0/2
  double tgy1[2], tgy3[2], tgx0[2], tgx2[2];
  {
    const double* blk = sY + tl<N, 3>(el, a, 0);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double s1 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double y = blk[c * N + i];
        s1 += C.eR[i] * y;
        s3 += C.eL[i] * y;
      }
      tgy1[c] = s1;
      tgy3[c] = s3;
    }
    const double* bx = sX + tl<N, 3>(el, a, 0);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double s0 = 0.0, s2 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double x = bx[c * N + i];
        s2 += C.eR[i] * x;
        s0 += C.eL[i] * x;
      }
      tgx2[c] = s2;
      tgx0[c] = s0;
    }
  }
  // q traces on faces 0 (point a) and 2 (point N-1-a) from column a
  double t0q[4] = {0, 0, 0, 0}, t2q[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x[4];
    lds4(sQ + ((el * N + i) * N + a) * 4, x);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      t2q[v] += C.eR[i] * x[v];
      t0q[v] += C.eL[i] * x[v];
    }
  }
  // one-sided viscous normal fluxes (spatial.py:456-464) into the face
  // records: face 1 +fx, face 3 -fx, face 2 +fy, face 0 -fy
  double o[4];
  {
    const double gyv[2] = {tgy1[0], tgy1[1]};
    visc_fx(t1q, tgx1, gyv, ph, o);
    stg4_last(frec + (int64_t)ri[1] * FREC4 + (lft[1] ? 4 : 8), o);
  }
  {
    const double gyv[2] = {tgy3[0], tgy3[1]};
    visc_fx(t3q, tgx3, gyv, ph, o);
    o[1] = -o[1], o[2] = -o[2], o[3] = -o[3];
    stg4_last(frec + (int64_t)ri[3] * FREC4 + (lft[3] ? 4 : 8), o);
  }
  {
    const double gxv[2] = {tgx2[0], tgx2[1]};
    visc_fy(t2q, gxv, tgy2, ph, o);
    stg4_last(frec + (int64_t)ri[2] * FREC4 + (lft[2] ? 4 : 8), o);
  }
  {
    const double gxv[2] = {tgx0[0], tgx0[1]};
    visc_fy(t0q, gxv, tgy0, ph, o);
    o[1] = -o[1], o[2] = -o[2], o[3] = -o[3];
    stg4_last(frec + (int64_t)ri[0] * FREC4 + (lft[0] ? 4 : 8), o);
  }
}

// ---------------------------------------------------------------------------
// The common total normal flux of the two-kernel chain, split by side
// (spatial.py:559-568; BR1: Fc = F - (fl - fr)/2 = (F - fl/2) + fr/2; LDG:
// Fc = F + fr; boundary: Fc = F - fl, energy row kept on adiabatic walls)
__device__ __forceinline__ void gh_left(const Phys& ph, bool bnd, int tag, const double* F, const double* fl,
                                        double* G) {
  if (bnd) {
#pragma unroll
    for (int v = 0; v < 4; ++v) G[v] = F[v] - ((v == 3 && tag == T_WALL_ADIABATIC) ? 0.0 : fl[v]);
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v) G[v] = ph.ldg ? F[v] : F[v] - 0.5 * fl[v];
  }
}
__device__ __forceinline__ void gh_right(const Phys& ph, const double* fr, double* H) {
  H[0] = ph.ldg ? fr[1] : 0.5 * fr[1];
  H[1] = ph.ldg ? fr[2] : 0.5 * fr[2];
  H[2] = ph.ldg ? fr[3] : 0.5 * fr[3];
  H[3] = 0.0;
}
// Fc on the own normal from the record halves (H = zeros on boundary faces)
__device__ __forceinline__ void gh_combine(bool lft, const double* G, const double* H, double* Fc) {
  const double c0 = G[0], c1 = G[1] + H[0], c2 = G[2] + H[1], c3 = G[3] + H[2];
  Fc[0] = lft ? c0 : -c0;
  Fc[1] = lft ? c1 : -c1;
  Fc[2] = lft ? c2 : -c2;
  Fc[3] = lft ? c3 : -c3;
}

// offset (doubles) of face-point record ri = slot * N + k and the stride
// between its parts: point by point, or (NS two-kernel chain, RSOA) part by part
template <int N>
__device__ __forceinline__ int64_t rec_off(int ri, bool soa) {
  return soa ? (int64_t)(ri / N) * (N * FREC) + (ri % N) * 4 : (int64_t)ri * FREC;
}
// One face record as a thread of the two-kernel chain holds it
struct FaceRec {
  double a[4], b[4];   // REC12: F, fl;  else G, H
#if PMGB_RECT_REC12
  double c[4];         // fr
#endif
};
__device__ __forceinline__ void rec_load(const double* rec, bool visc, bool interior, bool lv, FaceRec& r,
                                         int ps = 4) {
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    r.a[v] = r.b[v] = 0.0;
#if PMGB_RECT_REC12
    r.c[v] = 0.0;
#endif
  }
  if (!lv) return;
  ldg4c(rec, r.a);
#if PMGB_RECT_REC12
  if (visc) {
    ldg4c(rec + ps, r.b);
    if (interior) ldg4c(rec + 2 * ps, r.c);
  }
#else
  if (visc && interior) ldg4c(rec + 4, r.b);
#endif
}
// Fc on the thread's own normal (k_rfc's arithmetic when REC12)
__device__ __forceinline__ void rec_combine(const Phys& ph, bool visc, bool bnd, int tag, bool lft, const FaceRec& r,
                                            double* Fc) {
#if PMGB_RECT_REC12
  double c[4] = {r.a[0], r.a[1], r.a[2], r.a[3]};
  if (visc) {
    double Fv[4];
    if (bnd) {
#pragma unroll
      for (int v = 0; v < 4; ++v) Fv[v] = common_fv(ph, false, true, r.b[v], r.b[v]);
      if (tag == T_WALL_ADIABATIC) Fv[3] = 0.0;
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) Fv[v] = common_fv(ph, true, true, r.b[v], r.c[v]);
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) c[v] = c[v] - Fv[v];
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) Fc[v] = lft ? c[v] : -c[v];
#else
  gh_combine(lft, r.a, r.b, Fc);
#endif
}
// k_rgf's side of the record: F and the one-sided viscous flux o on the own normal
__device__ __forceinline__ void rec_put(const Phys& ph, bool bnd, int tag, bool lft, const double* F, const double* o,
                                        double* rec, int ps = 4) {
#if PMGB_RECT_REC12
  if (lft) {
    stg4_last(rec, F);
    stg4_last(rec + ps, o);
  } else {
    stg4_last(rec + 2 * ps, o);
  }
#else
  double r[4];
  if (lft) {
    gh_left(ph, bnd, tag, F, o, r);
    stg4_last(rec, r);
  } else {
    gh_right(ph, o, r);
    stg4_last(rec + 4, r);
  }
#endif
}

// ---------------------------------------------------------------------------
// Static face data of line thread (el, a): its four face points sit at the
// ends of row a (faces 1, 3) and of column a (faces 2, 0).
struct FaceStat {
  int ri[4];     // face-record index: unique face slot * N + L's point
  int nb[4];     // neighbour element (-1: boundary face)
  int fl[4];     // the link flags {neighbour face, rev, is_left, tag}
};
template <int N>
__device__ __forceinline__ void face_stat(const RectMesh& m, int64_t e, int a, bool live, FaceStat& s) {
#pragma unroll
  for (int f = 0; f < 4; ++f) s.ri[f] = 0, s.nb[f] = -1, s.fl[f] = 8;
  if (!live) return;
  const int4 sl = __ldg(reinterpret_cast<const int4*>(m.fslot) + e);
  const int4 l01 = __ldg(reinterpret_cast<const int4*>(m.link) + 2 * e);
  const int4 l23 = __ldg(reinterpret_cast<const int4*>(m.link) + 2 * e + 1);
  const int slot[4] = {sl.x, sl.y, sl.z, sl.w};
  const int2 lk[4] = {make_int2(l01.x, l01.y), make_int2(l01.z, l01.w), make_int2(l23.x, l23.y),
                      make_int2(l23.z, l23.w)};
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int k = (f >= 2) ? N - 1 - a : a;
    const bool lft = lk[f].x < 0 || lk_left(lk[f].y);
    const int kL = (!lft && lk_rev(lk[f].y)) ? N - 1 - k : k;
    s.ri[f] = slot[f] * N + kL;
    s.nb[f] = lk[f].x;
    s.fl[f] = lk[f].y;
  }
}

// ---------------------------------------------------------------------------
// k_rgf (NS kinds): k_rface and k_rgrad in one element kernel.  The own
// traces come from the staged q block; only the neighbours' traces are
// gathered (issued before the q block is awaited).  Every thread forms the
// common value What of its four face points (both sides of a face evaluate
// the same expression on the same operands), the side that owns a face (L)
// evaluates the interface flux once, and What goes to the element's own
// What block only -- no What round trip inside this kernel, no scattered
// What stores.  Bitwise the results of k_rface + k_rgrad.

template <int P, bool HASX> struct GFL {
  using R = RC<P>;
  static constexpr int BUF = R::EPB * TL<R::N, 3>::S;
  static constexpr int A = 2 * BUF, B = HASX ? R::QD : 0;
  static constexpr int STAGE = A > B ? A : B;
  static constexpr int OFF_BAR = R::QD + STAGE;
  static constexpr bool WTMA = PMGB_RECT_WTMA >= 0 ? PMGB_RECT_WTMA != 0 : (P == 4 && !HASX);
  static constexpr int OFF_WS = OFF_BAR + 2;   // What block staged for the bulk store (WTMA)
  static constexpr size_t BYTES = sizeof(double) * (OFF_BAR + 2 + (WTMA ? R::WD : 0));
};

template <int P, int KIND, bool HASX>
__global__ void __launch_bounds__(RC<P>::TH, RC<P>::MINB)
k_rgf(const FrConst C, const RectMesh m, const double* __restrict__ q, const double* __restrict__ X, double eps,
      double* __restrict__ wh, double* __restrict__ frec, int* __restrict__ bad) {
  using R = RC<P>;
  using L = GFL<P, HASX>;
  constexpr bool RSOA = PMGB_RECT_RSOA && PMGB_RECT_REC12;
  constexpr int N = R::N, NP = R::NP, E = R::EPB;
  extern __shared__ __align__(128) double sm[];
  double* sQ = sm;
  double* sX = sm + R::QD;            // X block; then W, then gx (column blocks)
  double* sY = sm + R::QD + L::BUF;   // gy (row blocks)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  const int t = threadIdx.x;
  const int el = t / N, a = t % N;  // row a of element el; also column a
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int ne = (int)((m.M - e0) < E ? (m.M - e0) : E);
  const int64_t e = e0 + el;
  const bool live = t < E * N && el < ne;
  const Phys ph = phys_of(C);
  const double g = C.gamma;
  if (t == 0) mbar_init(bar);
  __syncthreads();
  // the stream predecessor (launched ahead of with programmatic
  // serialization) may still be writing q or reading What / the records
  pdl_wait();
  pdl_trigger();
  stage_q<P, HASX, false>(sQ, sX, q, X, e0, ne, bar);
#if PMGB_RECT_PF > 0
  if (t == 32 && ((int64_t)blockIdx.x + PMGB_RECT_PF + 1) * E <= m.M)
    l2_prefetch(q + ((int64_t)blockIdx.x + PMGB_RECT_PF) * E * NP * 4, (uint32_t)E * NP * 32);
#endif
  FaceStat fs;
  face_stat<N>(m, e, a, live, fs);
  const double2 rg = live ? __ldg(m.rgeo + e) : make_double2(0.0, 0.0);
  // the neighbours' traces at the thread's four face points, gathered
  // from q (issued before the q block is awaited)
  double qn[4][4];
  double2 nrm[4];
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    qn[f][0] = qn[f][1] = qn[f][2] = qn[f][3] = 1.0;
    nrm[f] = make_double2(0.0, 0.0);
    if (live) {
      nrm[f] = __ldg(reinterpret_cast<const double2*>(m.geom + e * 20 + 8 + 2 * f));
      constexpr bool NBS = R::NBS == 2 || (R::NBS == 1 && HASX);
      const bool ins = NBS && fs.nb[f] >= e0 && fs.nb[f] < e0 + ne;
      if (fs.nb[f] >= 0 && !ins) {
        const int k = (f >= 2) ? N - 1 - a : a;
        face_trace<P, HASX>(C, q, X, eps, fs.nb[f], lk_face(fs.fl[f]), lk_rev(fs.fl[f]) ? N - 1 - k : k, qn[f]);
      }
    }
  }
  mbar_wait(bar, 0);
  if constexpr (HASX) {
    form_qp_rows<P>(sQ, sX, eps, ne);
    __syncthreads();
  }
  if constexpr (R::NBS == 2 || (R::NBS == 1 && HASX)) {
#pragma unroll
    for (int f = 0; f < 4; ++f)
      if (live && fs.nb[f] >= e0 && fs.nb[f] < e0 + ne) {
        const int k = (f >= 2) ? N - 1 - a : a;
        face_trace_s<P>(C, sQ, (int)(fs.nb[f] - e0), lk_face(fs.fl[f]), lk_rev(fs.fl[f]) ? N - 1 - k : k, qn[f]);
      }
  }
  // own traces: faces 1 / 3 from row a, faces 2 / 0 from column a
  double qo[4][4];
#pragma unroll
  for (int f = 0; f < 4; ++f) qo[f][0] = qo[f][1] = qo[f][2] = qo[f][3] = 0.0;
  const double* row = sQ + (el * N + a) * R::RS;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x[4];
    lds4(row + 4 * i, x);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      qo[1][v] += C.eR[i] * x[v];
      qo[3][v] += C.eL[i] * x[v];
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x[4];
    lds4(sQ + (el * N + i) * R::RS + a * 4, x);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      qo[2][v] += C.eR[i] * x[v];
      qo[0][v] += C.eL[i] * x[v];
    }
  }
  // common values; the interface flux on the faces this element owns
  double whv[4][3], uv[4][2], Fk[4][4];
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const bool bnd = fs.nb[f] < 0;
    const bool lft = bnd || lk_left(fs.fl[f]);
    const int tag = lk_tag(fs.fl[f]);
    Fk[f][0] = Fk[f][1] = Fk[f][2] = Fk[f][3] = 0.0;
    const Pr O = prim_of(qo[f], g);
    uv[f][0] = O.u;
    uv[f][1] = O.v;
    double qc[4];
    if (bnd)
      ghost<KIND>(qo[f], tag, nrm[f].x, nrm[f].y, C.qinf, qc);
    else
      qc[0] = qn[f][0], qc[1] = qn[f][1], qc[2] = qn[f][2], qc[3] = qn[f][3];
    const Pr Q = prim_of(qc, g);
    double wo[3] = {O.u, O.v, O.p * O.ir}, wq[3] = {Q.u, Q.v, Q.p * Q.ir};
    if (lft) {
      if (live && bad != nullptr) {
        if (!(O.r > 0.0 && O.p > 0.0)) atomicMin(bad + 1, (int)e);
        if (!bnd && !(Q.r > 0.0 && Q.p > 0.0)) atomicMin(bad + 1, fs.nb[f]);
      }
      if (ph.riemann)
        rusanov_pr(qo[f], O, qc, Q, nrm[f].x, nrm[f].y, g, Fk[f]);
      else
        roe_pr(qo[f], O, qc, Q, nrm[f].x, nrm[f].y, g, Fk[f]);
      if (bnd) ghost_w<KIND>(ph, tag, wo, wq);
#pragma unroll
      for (int c = 0; c < 3; ++c) whv[f][c] = common_w(ph, !bnd, true, wo[c], wq[c]);
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) whv[f][c] = common_w(ph, true, true, wq[c], wo[c]);
    }
    if (live) {
      if constexpr (L::WTMA) {
        double* dw = sm + L::OFF_WS + ((el * 4 + f) * N + ((f >= 2) ? N - 1 - a : a)) * 3;
        dw[0] = whv[f][0], dw[1] = whv[f][1], dw[2] = whv[f][2];
      } else {
        double* dw = wh + ((e * 4 + f) * N + ((f >= 2) ? N - 1 - a : a)) * 3;
        stg1_last(dw, whv[f][0]), stg1_last(dw + 1, whv[f][1]), stg1_last(dw + 2, whv[f][2]);
      }
    }
  }
  if constexpr (L::WTMA) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  // rows: primitives, W
  double w[3][N];
  {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double x[4];
      lds4(row + 4 * i, x);
      const Pr s = prim_of(x, g);
      ok = ok && (s.r > 0.0) && (s.p > 0.0);
      w[0][i] = s.u;
      w[1][i] = s.v;
      w[2][i] = s.p * s.ir;
    }
    if (live && !ok && bad != nullptr) atomicMin(bad, (int)e);
  }
  // W into column blocks: block (el, i) holds column i, [c][row]
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) sX[tl<N, 3>(el, i, c * N + a)] = w[c][i];
  // gx along row a (faces 1 and 3)
  double gx[3][N];
  line_gradient<N>(C, w, whv[1], whv[3], rg.x, gx);
  __syncthreads();
  if constexpr (L::WTMA) {
    if (t == 0) {   // the staged What block is complete: one bulk store
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(wh + e0 * 4 * N * 3),
                   "r"(saddr(sm + L::OFF_WS)), "r"((uint32_t)ne * 4 * N * 24)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  // column a: W of the column, gy (faces 2 and 0)
  double gy[3][N];
  {
    const double* blk = sX + tl<N, 3>(el, a, 0);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int i = 0; i < N; ++i) w[c][i] = blk[c * N + i];
    line_gradient<N>(C, w, whv[2], whv[0], rg.y, gy);
  }
  __syncthreads();  // W reads done
  // gx rows -> column blocks of sX; gy columns -> row blocks of sY
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      sX[tl<N, 3>(el, i, c * N + a)] = gx[c][i];
      sY[tl<N, 3>(el, i, c * N + a)] = gy[c][i];
    }
  // traces of the own-line components: gx on faces 1/3, gy on faces 0/2
  double tgx1[3], tgx3[3], tgy0[3], tgy2[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double s1 = 0.0, s3 = 0.0, s0 = 0.0, s2 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s1 += C.eR[i] * gx[c][i];
      s3 += C.eL[i] * gx[c][i];
      s2 += C.eR[i] * gy[c][i];
      s0 += C.eL[i] * gy[c][i];
    }
    tgx1[c] = s1;
    tgx3[c] = s3;
    tgy2[c] = s2;
    tgy0[c] = s0;
  }
  __syncthreads();
  if (!live) return;
  // rows: gy along row a -> gy traces on faces 1/3; columns: gx -> faces 0/2
  double tgy1[2], tgy3[2], tgx0[2], tgx2[2];
  {
    const double* blk = sY + tl<N, 3>(el, a, 0);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double s1 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double y = blk[c * N + i];
        s1 += C.eR[i] * y;
        s3 += C.eL[i] * y;
      }
      tgy1[c] = s1;
      tgy3[c] = s3;
    }
    const double* bx = sX + tl<N, 3>(el, a, 0);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double s0 = 0.0, s2 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double x = bx[c * N + i];
        s2 += C.eR[i] * x;
        s0 += C.eL[i] * x;
      }
      tgx2[c] = s2;
      tgx0[c] = s0;
    }
  }
  // one-sided viscous normal fluxes (spatial.py:456-464): face 1 +fx, face 3
  // -fx, face 2 +fy, face 0 -fy; each side's half of the face record
  auto put = [&](int f, double* o) {
    const bool bnd = fs.nb[f] < 0;
    rec_put(ph, bnd, lk_tag(fs.fl[f]), bnd || lk_left(fs.fl[f]), Fk[f], o, frec + rec_off<N>(fs.ri[f], RSOA),
            RSOA ? 4 * N : 4);
  };
  double o[4];
  {
    const double gyv[2] = {tgy1[0], tgy1[1]};
    visc_fx_uv(uv[1][0], uv[1][1], tgx1, gyv, ph, o);
    put(1, o);
  }
  {
    const double gyv[2] = {tgy3[0], tgy3[1]};
    visc_fx_uv(uv[3][0], uv[3][1], tgx3, gyv, ph, o);
    o[1] = -o[1], o[2] = -o[2], o[3] = -o[3];
    put(3, o);
  }
  {
    const double gxv[2] = {tgx2[0], tgx2[1]};
    visc_fy_uv(uv[2][0], uv[2][1], gxv, tgy2, ph, o);
    put(2, o);
  }
  {
    const double gxv[2] = {tgx0[0], tgx0[1]};
    visc_fy_uv(uv[0][0], uv[0][1], gxv, tgy0, ph, o);
    o[1] = -o[1], o[2] = -o[2], o[3] = -o[3];
    put(0, o);
  }
  if constexpr (L::WTMA) {
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// ---------------------------------------------------------------------------
// k_rasm: point fluxes, FR divergence, fused epilogue

// FOLD: no Fc block -- the thread gathers its four face records and forms
// the common flux itself (k_rfc folded in)
template <int P, int KIND, bool HASX, bool FOLD = false> struct AL {
  using R = RC<P>;
  static constexpr bool VISC = KT<KIND>::VISC;
  static constexpr int S_ = TL<R::N, 3>::S > TL<R::N, 4>::S ? TL<R::N, 3>::S : TL<R::N, 4>::S;
  static constexpr int BUF = R::EPB * S_;
  static constexpr int WD = VISC ? R::WD : 0;
  static constexpr int FD = FOLD ? 0 : R::FD;
  static constexpr int A = 2 * BUF, B = WD + FD + (HASX ? R::QD : 0);
  static constexpr int STAGE = A > B ? A : B;
  static constexpr int OFF_F = R::QD + STAGE - FD, OFF_W = OFF_F - WD, OFF_BAR = R::QD + STAGE;
  static constexpr size_t BYTES = sizeof(double) * (OFF_BAR + 2);
};

template <int P, int KIND, int EK, bool HASX, bool FOLD = false>
__global__ void __launch_bounds__(RC<P>::TH, RC<P>::MINB)
k_rasm(const FrConst C, const RectMesh m, const double* __restrict__ q, const double* __restrict__ X, double eps,
       const double* __restrict__ wh, const double* __restrict__ fc, const Epi ep, double* __restrict__ out,
       int* bad, Status* st) {
  using R = RC<P>;
  using L = AL<P, KIND, HASX, FOLD>;
  constexpr int N = R::N, NP = R::NP, E = R::EPB;
  constexpr bool VISC = KT<KIND>::VISC;
  constexpr bool RSOA = PMGB_RECT_RSOA && PMGB_RECT_REC12 && VISC && FOLD;
  extern __shared__ __align__(128) double sm[];
  double* sQ = sm;
  double* sX = sm + R::QD;            // X block; then W, then fy (column blocks)
  double* sY = sm + R::QD + L::BUF;   // gy (row blocks), then X_xi (column blocks)
  const double* sWb = sm + L::OFF_W;  // What block [el][f][k][3]
  const double* sFb = sm + L::OFF_F;  // Fc block [el][f][k][4]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  const int t = threadIdx.x;
  const int el = t / N, a = t % N;
  // FOLD chain: element blocks in descending order -- the blocks the
  // previous kernel touched last (its q reads, its What / record writes)
  // are the ones still in L2
  const int64_t blk = (FOLD && PMGB_RECT_REV) ? (int64_t)gridDim.x - 1 - blockIdx.x : (int64_t)blockIdx.x;
  const int64_t e0 = blk * E;
  const int ne = (int)((m.M - e0) < E ? (m.M - e0) : E);
  const int64_t e = e0 + el;
  const bool live = t < E * N && el < ne;
  const Phys ph = phys_of(C);
  const double g = C.gamma;
  if (t == 0) {
    mbar_init(bar);
    mbar_init(bar + 1);
  }
  __syncthreads();
  const uint32_t qbytes = (uint32_t)ne * NP * 32;
  stage_q<P, HASX, true>(sQ, sX, q, X, e0, ne, bar);
#if PMGB_RECT_EPF
  if (t == 32) epi_prefetch<EK>(ep, e0 * NP * 4, qbytes);
#endif
  const double2 rg = live ? __ldg(m.rgeo + e) : make_double2(1.0, 1.0);
  FaceStat fs;
  if constexpr (FOLD) face_stat<N>(m, e, a, live, fs);
  pdl_wait();  // What and the face records (k_rface / k_rgf; Fc: k_rfc), status flags
  if (t == 0) {
    const uint32_t fb = FOLD ? 0u : (uint32_t)ne * 4 * N * 32, wb = (uint32_t)ne * 4 * N * 24;
    if (VISC || !FOLD) mbar_expect(bar + 1, VISC ? fb + wb : fb);
    if (!FOLD) bulk_g2s_first(sm + L::OFF_F, fc + e0 * 4 * N * 4, fb, bar + 1);
    if (VISC) bulk_g2s_first(sm + L::OFF_W, wh + e0 * 4 * N * 3, wb, bar + 1);
    if (blockIdx.x == 0) commit_status(bad, st);
  }
  double fcv[4][4];
  FaceRec rc[4];
  if constexpr (FOLD) {
    // the four face records (fc here is the face-record array), gathered
    // while the q block is in flight
#pragma unroll
    for (int f = 0; f < 4; ++f)
      rec_load(fc + rec_off<N>(fs.ri[f], RSOA), VISC, fs.nb[f] >= 0, live, rc[f], RSOA ? 4 * N : 4);
  }
#if PMGB_RECT_PF > 0   // the q / What blocks of the CTA PMGB_RECT_PF positions later in the walk
  {
    const int64_t bn = (FOLD && PMGB_RECT_REV) ? blk - PMGB_RECT_PF : blk + PMGB_RECT_PF;
    if (t == 32 && bn >= 0 && (bn + 1) * E <= m.M) {
      l2_prefetch(q + bn * E * NP * 4, (uint32_t)E * NP * 32);
      if (VISC) l2_prefetch(wh + bn * E * 4 * N * 3, (uint32_t)E * 4 * N * 24);
    }
  }
#endif
  auto combine = [&]() {
#pragma unroll
    for (int f = 0; f < 4; ++f)
      rec_combine(ph, VISC, fs.nb[f] < 0, lk_tag(fs.fl[f]), fs.nb[f] < 0 || lk_left(fs.fl[f]), rc[f], fcv[f]);
  };
  mbar_wait(bar, 0);
  if constexpr (HASX) {
    form_qp_rows<P>(sQ, sX, eps, ne);
    __syncthreads();
  }
  const double* row = sQ + (el * N + a) * R::RS;
  double w[3][N];
  if constexpr (VISC) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double x[4];
      lds4(row + 4 * i, x);
      const Pr s = prim_of(x, g);
      w[0][i] = s.u;
      w[1][i] = s.v;
      w[2][i] = s.p * s.ir;
    }
  }
  if constexpr (FOLD) combine();
  if constexpr (VISC || !FOLD) mbar_wait(bar + 1, 0);
  double whv[4][3];
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int fp = el * 4 * N + fpt_of<N>(f, a);
    if constexpr (VISC) {
#pragma unroll
      for (int c = 0; c < 3; ++c) whv[f][c] = sWb[fp * 3 + c];
    }
    if constexpr (!FOLD) lds4(sFb + fp * 4, fcv[f]);
  }
  __syncthreads();  // the stage (X, What, Fc blocks) is free
  double gy[3][N];
  if constexpr (VISC) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < 3; ++c) sX[tl<N, 3>(el, i, c * N + a)] = w[c][i];
    __syncthreads();
    // column a: gy -> row blocks
    {
      const double* blk = sX + tl<N, 3>(el, a, 0);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int i = 0; i < N; ++i) w[c][i] = blk[c * N + i];
      double gc[3][N];
      line_gradient<N>(C, w, whv[2], whv[0], rg.y, gc);
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) sY[tl<N, 3>(el, i, c * N + a)] = gc[c][i];
    }
    __syncthreads();
    const double* blk = sY + tl<N, 3>(el, a, 0);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int i = 0; i < N; ++i) gy[c][i] = blk[c * N + i];
  }
  // row a: primitives (again: cheaper than holding them through the column
  // pass), gx, point fluxes -- fx stays in registers, fy -> column blocks
  double qr[4][N];
  Pr pr[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x[4];
    lds4(row + 4 * i, x);
#pragma unroll
    for (int v = 0; v < 4; ++v) qr[v][i] = x[v];
    pr[i] = prim_of(x, g);
  }
  double gx[3][N];
  if constexpr (VISC) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      w[0][i] = pr[i].u;
      w[1][i] = pr[i].v;
      w[2][i] = pr[i].p * pr[i].ir;
    }
    line_gradient<N>(C, w, whv[1], whv[3], rg.x, gx);
  }
  double fx[4][N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const Pr& s = pr[i];
    double Fx[4], Fy[4];
    Fx[0] = qr[1][i];
    Fx[1] = qr[1][i] * s.u + s.p;
    Fx[2] = qr[1][i] * s.v;
    Fx[3] = s.u * (qr[3][i] + s.p);
    Fy[0] = qr[2][i];
    Fy[1] = qr[2][i] * s.u;
    Fy[2] = qr[2][i] * s.v + s.p;
    Fy[3] = s.v * (qr[3][i] + s.p);
    if constexpr (VISC) {
      const double gxx[3] = {gx[0][i], gx[1][i], gx[2][i]};
      const double gyy[3] = {gy[0][i], gy[1][i], gy[2][i]};
      const double d = gxx[0] + gyy[1];
      const double txx = ph.mu * (2.0 * gxx[0] - (2.0 / 3.0) * d);
      const double tyy = ph.mu * (2.0 * gyy[1] - (2.0 / 3.0) * d);
      const double txy = ph.mu * (gyy[0] + gxx[1]);
      Fx[1] = Fx[1] - txx;
      Fx[2] = Fx[2] - txy;
      Fx[3] = Fx[3] - (s.u * txx + s.v * txy + ph.kappa * gxx[2]);
      Fy[1] = Fy[1] - txy;
      Fy[2] = Fy[2] - tyy;
      Fy[3] = Fy[3] - (s.u * txy + s.v * tyy + ph.kappa * gyy[2]);
      Fx[0] = Fx[0] - 0.0;
      Fy[0] = Fy[0] - 0.0;
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      fx[v][i] = Fx[v];
      sX[tl<N, 4>(el, i, v * N + a)] = Fy[v];
    }
  }
  // X_xi along row a
  double xx[4][N];
  line_div<N>(C, fx, fcv[1], fcv[3], xx);
  if constexpr (VISC) __syncthreads();  // gy row reads of sY done
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v) sY[tl<N, 4>(el, i, v * N + a)] = xx[v][i];
  __syncthreads();
  if (!live) return;
  // column a: fy and X_xi of the column, faces 2 / 0, X_eta, R, epilogue.
  // The epilogue operands of point i + EPD are requested before point i is
  // formed and stored (the first EPD points before the column pass), so
  // their latency overlaps the arithmetic instead of heading every point.
  constexpr int EPD = (EK == EPI_R) ? 0 : (PMGB_RECT_EPD < N ? PMGB_RECT_EPD : N);
  double o1[N][4], o2[N][4], o3[N][4];
  auto epi_req = [&](int i) { epi_load4_k<EK>(ep, (e * NP + i * N + a) * 4, o1[i], o2[i], o3[i]); };
#pragma unroll
  for (int i = 0; i < EPD; ++i) epi_req(i);
  double fyc[4][N];
  {
    const double* blk = sX + tl<N, 4>(el, a, 0);
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int i = 0; i < N; ++i) fyc[v][i] = blk[v * N + i];
  }
  double xe[4][N];
  line_div<N>(C, fyc, fcv[2], fcv[0], xe);
  const double* bx = sY + tl<N, 4>(el, a, 0);
  constexpr bool NEEDQ = !(EK == EPI_R || EK == EPI_JV || EK == EPI_NEG_R);
  const double ce = (EK == EPI_RK) ? epi_rk_coef(ep, e) : 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {   // point (i, a)
    const int64_t pt = e * NP + i * N + a;
    double qv[4] = {0, 0, 0, 0};
    if constexpr (NEEDQ) lds4(sQ + (el * N + i) * R::RS + a * 4, qv);
    double o[4];
    if constexpr (EK != EPI_R)
      if (i + EPD < N) epi_req(i + EPD);   // operands as 256-bit loads
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double Rv = -(rg.x * bx[v * N + i] + rg.y * xe[v][i]);
      if constexpr (EK == EPI_R)
        o[v] = Rv;
      else
        o[v] = (EK == EPI_RK) ? epi_rk(ep, ce, Rv, qv[v], o1[i][v], o2[i][v], o3[i][v])
                              : epi_pre_k<EK>(ep, Rv, qv[v], o1[i][v], o2[i][v], o3[i][v]);
    }
    stg4_first(out + pt * 4, o);
  }
}

// ---------------------------------------------------------------------------
// host side

template <typename... KArgs, typename... Args>
static void launch_pdl_r(void (*kernel)(KArgs...), unsigned grid, int threads, size_t smem, cudaStream_t st,
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

using RasmFn = void (*)(const FrConst, const RectMesh, const double*, const double*, double, const double*,
                        const double*, const Epi, double*, int*, Status*);

template <int P, int KIND, bool HASX, bool FOLD>
static RasmFn rasm_for(int mode) {
  switch (mode) {
    case EPI_R: return k_rasm<P, KIND, EPI_R, HASX, FOLD>;
    case EPI_JV: return k_rasm<P, KIND, EPI_JV, HASX, FOLD>;
    case EPI_STAGE_JV: return k_rasm<P, KIND, EPI_STAGE_JV, HASX, FOLD>;
    case EPI_DEFECT: return k_rasm<P, KIND, EPI_DEFECT, HASX, FOLD>;
    case EPI_F: return k_rasm<P, KIND, EPI_F, HASX, FOLD>;
    case EPI_RK: return k_rasm<P, KIND, EPI_RK, HASX, FOLD>;
  }
  return k_rasm<P, KIND, -1, HASX, FOLD>;
}

template <int P, int KIND, bool HASX>
static void set_rect_attrs() {
  for (int md : {(int)EPI_R, (int)EPI_JV, (int)EPI_STAGE_JV, (int)EPI_DEFECT, (int)EPI_F, (int)EPI_RK, -1}) {
    cudaFuncSetAttribute(rasm_for<P, KIND, HASX, false>(md), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)AL<P, KIND, HASX, false>::BYTES);
    cudaFuncSetAttribute(rasm_for<P, KIND, HASX, true>(md), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)AL<P, KIND, HASX, true>::BYTES);
  }
  if constexpr (KT<KIND>::VISC) {
    cudaFuncSetAttribute(k_rgrad<P, HASX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GL<P, HASX>::BYTES);
    cudaFuncSetAttribute(k_rgf<P, KIND, HASX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)GFL<P, HASX>::BYTES);
  }
}

// d.has_rect: 3 the two-kernel chain k_rgf / k_rface + k_rasm (common flux
// folded in), 2 the four-kernel chain it replaced, 1 the faster of the two
// at this degree: the four-kernel chain at p = 2 (config-2 coarse level R
// 55.4 vs 63.8 us), the two-kernel chain elsewhere (p = 1: 34.7 vs 39.0,
// p = 3: 85.8 vs 102.7, p = 4: 105.1 vs 114.8, p = 5: even;
// profiles/r2/ab_chain_r2u.log).  Measured slower and removed: a
// persistent, double-buffered k_rasm (profiles/r2/ab_chain_r2m.jsonl,
// "rect2p") and a shared-memory hand-over of the traces between
// neighbours of one CTA in k_rgf (profiles/r2/ab_xch_r2n.log).
template <int P> constexpr bool rect_two_kernel_default() { return P != 2; }
#ifndef PMGB_RECT_PDL0   // measured: config-2 R 113.0 -> 110.7 us, config 3 34.1 -> 32.0 us
#define PMGB_RECT_PDL0 1
#endif
template <int P, int KIND>
static int run_rect(const RectDev& rd, const DiscDev& d, const double* q, const double* X, double eps,
                    const Epi& epi, double* out, int* bad, Status* stp, cudaStream_t st) {
  using R = RC<P>;
  static std::atomic<unsigned long long> attr_seen{0};
  once_per_device(attr_seen, [&] {
    set_rect_attrs<P, KIND, false>();
    set_rect_attrs<P, KIND, true>();
  });
  const RectMesh m{d.M, rd.nface, rd.faces, rd.fslot, d.link, rd.rgeo, d.geom};
  const unsigned gf = (unsigned)((rd.nface * (P + 1) + 127) / 128);
  const unsigned ge = (unsigned)((d.M + R::EPB - 1) / R::EPB);
  const bool hx = X != nullptr;
  const bool fold = d.has_rect == 3 || (d.has_rect == 1 && rect_two_kernel_default<P>());
  if (fold && KT<KIND>::VISC) {
    if constexpr (KT<KIND>::VISC) {
#if PMGB_RECT_PDL0   // the chain's first kernel may start while its stream predecessor drains
      if (hx)
        launch_pdl_r(k_rgf<P, KIND, true>, ge, R::TH, GFL<P, true>::BYTES, st, d.C, m, q, X, eps, rd.wh, rd.frec,
                     bad);
      else
        launch_pdl_r(k_rgf<P, KIND, false>, ge, R::TH, GFL<P, false>::BYTES, st, d.C, m, q, X, eps, rd.wh,
                     rd.frec, bad);
#else
      if (hx)
        k_rgf<P, KIND, true><<<ge, R::TH, GFL<P, true>::BYTES, st>>>(d.C, m, q, X, eps, rd.wh, rd.frec, bad);
      else
        k_rgf<P, KIND, false><<<ge, R::TH, GFL<P, false>::BYTES, st>>>(d.C, m, q, X, eps, rd.wh, rd.frec, bad);
#endif
    }
  } else if (fold) {   // Euler kinds: F itself is the record's G
#if PMGB_RECT_PDL0
    if (hx)
      launch_pdl_r(k_rface<P, KIND, true, FREC>, gf, 128, 0, st, d.C, m, q, X, eps, rd.frec, rd.wh, bad);
    else
      launch_pdl_r(k_rface<P, KIND, false, FREC>, gf, 128, 0, st, d.C, m, q, X, eps, rd.frec, rd.wh, bad);
#else
    if (hx)
      k_rface<P, KIND, true, FREC><<<gf, 128, 0, st>>>(d.C, m, q, X, eps, rd.frec, rd.wh, bad);
    else
      k_rface<P, KIND, false, FREC><<<gf, 128, 0, st>>>(d.C, m, q, X, eps, rd.frec, rd.wh, bad);
#endif
  } else {
    if (hx)
      k_rface<P, KIND, true><<<gf, 128, 0, st>>>(d.C, m, q, X, eps, rd.frec, rd.wh, bad);
    else
      k_rface<P, KIND, false><<<gf, 128, 0, st>>>(d.C, m, q, X, eps, rd.frec, rd.wh, bad);
    if constexpr (KT<KIND>::VISC) {
      if (hx)
        launch_pdl_r(k_rgrad<P, true>, ge, R::TH, GL<P, true>::BYTES, st, d.C, m, q, X, eps,
                     (const double*)rd.wh, rd.frec, bad);
      else
        launch_pdl_r(k_rgrad<P, false>, ge, R::TH, GL<P, false>::BYTES, st, d.C, m, q, X, eps,
                     (const double*)rd.wh, rd.frec, bad);
    }
  }
  if (fold) {
    RasmFn fn = hx ? rasm_for<P, KIND, true, true>(epi.mode) : rasm_for<P, KIND, false, true>(epi.mode);
    const size_t smem = hx ? AL<P, KIND, true, true>::BYTES : AL<P, KIND, false, true>::BYTES;
    launch_pdl_r(fn, ge, R::TH, smem, st, d.C, m, q, X, eps, (const double*)rd.wh, (const double*)rd.frec, epi,
                 out, bad, stp);
    return (int)cudaGetLastError();
  }
  launch_pdl_r(k_rfc<P, KIND>, gf, 128, 0, st, d.C, m, (const double*)rd.frec, rd.fc);
  RasmFn fn = hx ? rasm_for<P, KIND, true, false>(epi.mode) : rasm_for<P, KIND, false, false>(epi.mode);
  const size_t smem = hx ? AL<P, KIND, true, false>::BYTES : AL<P, KIND, false, false>::BYTES;
  launch_pdl_r(fn, ge, R::TH, smem, st, d.C, m, q, X, eps, (const double*)rd.wh, (const double*)rd.fc, epi, out,
               bad, stp);
  return (int)cudaGetLastError();
}

int launch_residual_rect(const RectDev& rd, const DiscDev& d, const double* q, const double* X, double eps,
                         const Epi& epi, double* out, int* bad, Status* stp, cudaStream_t st) {
#ifdef PMGB_RECT_DEV   // experiment builds (tools/build_variant.sh): the config-2 / config-4 instances only
  switch (d.kind * 8 + d.p) {
    case K_NS * 8 + 3: return run_rect<3, K_NS>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_NS * 8 + 4: return run_rect<4, K_NS>(rd, d, q, X, eps, epi, out, bad, stp, st);
  }
  return -1000;
#else
  switch (d.kind * 8 + d.p) {
    case K_EULER * 8 + 1: return run_rect<1, K_EULER>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_EULER * 8 + 2: return run_rect<2, K_EULER>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_EULER * 8 + 3: return run_rect<3, K_EULER>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_EULER * 8 + 4: return run_rect<4, K_EULER>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_EULER * 8 + 5: return run_rect<5, K_EULER>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_NS * 8 + 1: return run_rect<1, K_NS>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_NS * 8 + 2: return run_rect<2, K_NS>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_NS * 8 + 3: return run_rect<3, K_NS>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_NS * 8 + 4: return run_rect<4, K_NS>(rd, d, q, X, eps, epi, out, bad, stp, st);
    case K_NS * 8 + 5: return run_rect<5, K_NS>(rd, d, q, X, eps, epi, out, bad, stp, st);
  }
  return -1000;
#endif
}

int rect_launches(const DiscDev& d, bool has_x) {
  (void)has_x;
  if (d.has_rect == 2 || (d.has_rect == 1 && d.p == 2)) return d.kind == K_NS ? 4 : 3;
  return 2;
}

bool rect_supported(int p, int kind) { return p >= 1 && p <= 5 && (kind == K_EULER || kind == K_NS); }

}  // namespace pmgb
