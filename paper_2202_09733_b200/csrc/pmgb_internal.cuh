// Internal definitions shared by the sm_100a FP64 kernels.
//
// Data layout in HBM (all FP64, element-major, reference AoS layout):
//   solution / residual vectors: [M][n][n][nv]   (eta index, xi index, var)
//     -- reference spatial.py:209-215, SURVEY Appendix B
//   face traces qtr:             [M][4][n][nv]   CCW point order per face
//   one-sided viscous flux fvn:  [M][4][n][nv]   along the element's own normal
//   geometry record:             [M][20]         see mesh.pack_geometry
//   face links:                  [M][4] int2     {nb elem | -1, flags}
//   EJ blocks / inverses:        [M][sz][sz] column-major (B^T row-major)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

namespace pmgb {

// Per-device one-time setup (kernel attributes are per device): runs f
// once for the current device and this flag word.  The bit is published
// only after f has run, under a lock, so a second host thread never
// launches before the attributes are set.
inline std::mutex& setup_mutex() {
  static std::mutex m;
  return m;
}
template <class F>
inline void once_per_device(std::atomic<unsigned long long>& seen, F&& f) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (seen.load(std::memory_order_acquire) & bit) return;
  std::lock_guard<std::mutex> lock(setup_mutex());
  if (seen.load(std::memory_order_acquire) & bit) return;
  f();
  seen.fetch_or(bit, std::memory_order_release);
}

enum Kind { K_EULER = 0, K_NS = 1, K_ADV = 2, K_ADVD = 3 };
enum Tag { T_WALL_ADIABATIC = 0, T_WALL_SLIP = 1, T_FAR_FIELD = 2, T_WALL_ISOTHERMAL = 3 };

// link.y bit layout
__host__ __device__ inline int lk_face(int y) { return y & 3; }
__host__ __device__ inline int lk_rev(int y) { return (y >> 2) & 1; }
__host__ __device__ inline int lk_left(int y) { return (y >> 3) & 1; }
__host__ __device__ inline int lk_tag(int y) { return (y >> 4) & 15; }

template <int KIND> struct KT;
template <> struct KT<K_EULER> { static constexpr int NV = 4, NW = 3; static constexpr bool VISC = false, FLOW = true; };
template <> struct KT<K_NS>    { static constexpr int NV = 4, NW = 3; static constexpr bool VISC = true,  FLOW = true; };
template <> struct KT<K_ADV>   { static constexpr int NV = 1, NW = 1; static constexpr bool VISC = false, FLOW = false; };
template <> struct KT<K_ADVD>  { static constexpr int NV = 1, NW = 1; static constexpr bool VISC = true,  FLOW = false; };

// CTA shape: one thread per solution point, EPB elements per CTA.
#ifndef PMGB_CTA_THREADS
#define PMGB_CTA_THREADS 128
#endif
#ifndef PMGB_CTA_THREADS_P5
#define PMGB_CTA_THREADS_P5 256
#endif
#ifndef PMGB_REG_TARGET_R   // R-only (EPI_R) instantiation of k_assemble_async
#define PMGB_REG_TARGET_R 72
#endif
#ifndef PMGB_BLOCKS_REGS   // k_blocks (FD element-block assembly)
#define PMGB_BLOCKS_REGS 80
#endif
#ifndef PMGB_REG_TARGET_R_P3
#define PMGB_REG_TARGET_R_P3 72
#endif
#ifndef PMGB_REG_TARGET_K_P3
#define PMGB_REG_TARGET_K_P3 72
#endif
#ifndef PMGB_REG_TARGET_R_P5   // p = 5 (256-thread CTAs)
#define PMGB_REG_TARGET_R_P5 64
#endif
#ifndef PMGB_REG_TARGET_K_P5
#define PMGB_REG_TARGET_K_P5 64
#endif
#ifndef PMGB_REG_TARGET_K   // the other compile-time epilogue modes
#define PMGB_REG_TARGET_K 72
#endif
#ifndef PMGB_REG_TARGET
#define PMGB_REG_TARGET 80
#endif
template <int P> struct BC {
  static constexpr int N = P + 1, NP = N * N, NF = 4 * N;
  static constexpr int THREADS = (P >= 5) ? PMGB_CTA_THREADS_P5 : PMGB_CTA_THREADS;
  static constexpr int EPB = (THREADS / NP) > 32 ? 32 : ((THREADS / NP) >= 1 ? THREADS / NP : 1);
};

// Operator matrices + physics constants, passed by value (constant bank).
struct FrConst {
  double D[36];               // D[k*n + i] = l_i'(x_k)
  double eL[6], eR[6], lL[6], lR[6], xg[6];
  double qinf[4];
  double gamma, mu, kappa, adv_x, adv_y, diff;
  double twall;  // T = p/rho on wall-isothermal faces (BASELINE option)
  int riemann;  // 0 Roe (reference), 1 Rusanov (BASELINE option)
  int ldg;      // 0 BR1 (reference), 1 LDG, C11 = 0, switch from the L element
};

struct FrMesh {
  int64_t M;
  const double* __restrict__ geom;  // (M,20)
  const int2* __restrict__ link;    // (M,4)
};

// Fused epilogue of the final residual phase (SURVEY 8(b) "fused prologue/epilogue").
enum EpiMode {
  EPI_R = 0,         // out = R(q)                                  spatial.py:501
  EPI_F = 1,         // out = s q - R(q)                            pmg.py:152-153
  EPI_DEFECT = 2,    // out = (Sb - (s q - R(q))) + Se              pmg.py:155-159
  EPI_JV = 3,        // out = s X - (R(q+eps X) - R0)/eps           newton_krylov.py:71-76
  EPI_STAGE_F = 4,   // out = (q - E)/adt - R(q)                    time_integration.py:138-141
  EPI_STAGE_JV = 5,  // out = X/dtau + (F(q+eps X) - Fk)/eps        newton_krylov.py:402-405
  EPI_NEG_R = 6,     // out = -R(q)       (steady stage function)   time_integration.py:139-140
  EPI_OUTER_F = 7,   // out = s q - R(q) - Se                       pmg.py:325-326
  EPI_RK = 8,        // out = Q0 + alpha dtau_e ((Sb - (s q - R)) + Se)   RK smoother stage
};

struct Epi {
  int mode;
  double s, eps, adt, dtau, sb_scalar, se_scalar;
  const double* X;    // perturbation direction (JV modes)
  const double* R0;   // R0 (EPI_JV) or Fk (EPI_STAGE_JV)
  const double* E;    // explicit stage part
  const double* Sb;   // S_base array (or null -> sb_scalar)
  const double* Se;   // S_extra array (or null -> se_scalar)
  const double* Q0;   // RK stage base state
  const double* dtau_e;  // RK per-element pseudo-time step (M)
  double alpha;          // RK stage coefficient
  int npe;            // dofs per element (set by the C ABI)
};

// Device-global status: first non-physical state seen since the last clear.
struct Status {
  int kind;             // 0 none, 1 state, 2 trace, 3 singular block
  int pad;
  long long element;
};

}  // namespace pmgb

// host-side launch helpers (defined in fr_kernels.cu etc.)
namespace pmgb {
// Rectangle fast path (fr_rect.cu): unique-face list and per-face records
struct RectDev {
  int64_t nface = 0;
  int4* faces = nullptr;    // {eL, fL | rev<<2 | bnd<<3 | tag<<4, eR, fR}
  int* fslot = nullptr;     // (M,4) face index of every element face
  double2* rgeo = nullptr;  // (M) {1/a0, 1/d0}
  double* frec = nullptr;   // (nface, n, 12): F (L normal), fvn of the L and R sides
  double* wh = nullptr;     // (M, 4, n, 3): BR1 common value What per element side
  double* fc = nullptr;     // (M, 4, n, 4): common total normal flux per element side
};

struct DiscDev {
  int p, kind;
  int64_t M;
  FrConst C;
  FrMesh mesh;
  double* geom;
  int2* link;
  double* qtr;   // scratch traces (M,4,n,nv)
  double* fvn;   // scratch viscous flux (M,4,n,nv)
  double* grad;  // scratch BR1 gradients, per CTA block in k_fvn's padded planes: [grid][2*nw][PS]
  double* qp;    // scratch perturbed state
  int nv;
  int64_t n_dofs;
  int has_rect = 0;  // every element an axis-aligned rectangle (fr_rect.cu)
  RectDev rect;
};

int launch_residual(const DiscDev& d, const double* q, const double* X, double eps,
                    const Epi& epi, double* out, cudaStream_t st);
int launch_residual_rect(const RectDev& rd, const DiscDev& d, const double* q, const double* X, double eps,
                         const Epi& epi, double* out, int* bad, Status* stp, cudaStream_t st);
bool rect_supported(int p, int kind);
int rect_launches(const DiscDev& d, bool has_x);  // kernels one evaluation launches on the rectangle path
size_t fr_grad_scratch_doubles(int p, int kind, int64_t M);
int launch_rk_lambda(const DiscDev& d, const double* q, double adv, double* lam, cudaStream_t st);
int launch_freeze(const DiscDev& d, const double* q, double* qtr, double* fvn, cudaStream_t st);
int launch_local_residual(const DiscDev& d, const int64_t* elems, int64_t B, const double* Q,
                          const double* qtr, const double* fvn, double* out, cudaStream_t st);
int launch_blocks(const DiscDev& d, const double* q, const double* qtr, const double* fvn,
                  double shift, double eps, double* blocksT, cudaStream_t st, const int* out_slot = nullptr);
int launch_coupling(const DiscDev& d, const double* q, const double* qtr, const double* fvn, double eps,
                    int64_t npairs, const int* pair_e, const signed char* pair_f, const int* pair_slot,
                    const signed char* pair_add, double* blocks, cudaStream_t st);
int launch_sparse_matvec(int64_t n_rows, int SZ, const int* indptr, const int* indices, const double* blocks,
                         const double* x, double* y, cudaStream_t st);
int launch_forces(const DiscDev& d, const double* q, int64_t nwall, const int* wall_e, const signed char* wall_f,
                  const double* weights, double* out, cudaStream_t st);
int status_clear_async(cudaStream_t st);
int status_read(cudaStream_t st, Status* out, int clear);
}  // namespace pmgb
