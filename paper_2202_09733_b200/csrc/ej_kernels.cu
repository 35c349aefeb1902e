// Element-Jacobi blocks: batched register-tiled Gauss-Jordan inversion and
// the HBM-bound batched block GEMV / fused EJ sweep update; pMG transfers.
//
// Reference: newton_krylov.py:187-210 (np.linalg.inv of the FD blocks,
// RuntimeError on a singular block), :157-171 (BlockJacobian.apply =
// einsum("mij,mj->mi")), pmg.py:162-164 (q <- q + omega B^-1 d),
// pmg.py:117-136 (Gamma (x) Gamma restriction, Pi (x) Pi prolongation).
//
// Inverse storage.  Gauss-Jordan runs in place with implicit partial
// pivoting (pivot of column k = largest |a_rk| over rows not yet used,
// ties to the lowest row -- the candidate set LAPACK getrf searches after
// its swaps), so rows never move.  The in-place result X satisfies
//     B^-1[i][j] = X[p_i][q_j],   p_k = pivot row of column k, q = p^-1,
// and is stored column-major XT[c][r] = X[r][c] with perm[0:sz] = p and
// perm[sz:2sz] = q (uint8).  The GEMV applies the permutations on the fly:
//     y[q_r] = sum_c XT[c][r] x[p_c]
// so nothing is ever un-permuted in memory.
#include <cstdlib>
#include <climits>
#include <cstdint>

#include "pmgb_internal.cuh"

namespace pmgb {

template <int SZ> struct GJTile;
template <> struct GJTile<1>   { static constexpr int TR = 1, TC = 1; };
template <> struct GJTile<4>   { static constexpr int TR = 1, TC = 2; };
template <> struct GJTile<9>   { static constexpr int TR = 3, TC = 3; };
template <> struct GJTile<16>  { static constexpr int TR = 2, TC = 4; };
template <> struct GJTile<25>  { static constexpr int TR = 5, TC = 5; };
template <> struct GJTile<36>  { static constexpr int TR = 3, TC = 6; };
template <> struct GJTile<64>  { static constexpr int TR = 4, TC = 8; };
#ifndef PMGB_GJ100_TR
#define PMGB_GJ100_TR 4
#endif
#ifndef PMGB_GJ100_TC
#define PMGB_GJ100_TC 10
#endif
template <> struct GJTile<100> { static constexpr int TR = PMGB_GJ100_TR, TC = PMGB_GJ100_TC; };
template <> struct GJTile<144> { static constexpr int TR = 8, TC = 6; };

template <int SZ> struct GJShape {
  static constexpr int TR = GJTile<SZ>::TR, TC = GJTile<SZ>::TC;
  static constexpr int NRG = (SZ + TR - 1) / TR, NCG = (SZ + TC - 1) / TC;
  static constexpr int THREADS = ((NRG * NCG + 31) / 32) * 32;
  static constexpr int ROWS_PER_LANE = (SZ + 31) / 32;
};

// One CTA per block.  BT: FD blocks, column-major (BT[c][r] = B[r][c]).
// Thread (rg, cg) holds a TR x TC register tile: rows rg + NRG i (row
// groups interleaved, so the warp's column-buffer reads are consecutive
// doubles: conflict-free), columns cg TC + j.  Per pivot step: column-k
// owners publish the column, every warp finds the pivot redundantly (lane
// l scans rows l + 32 m; max |a| over unused rows, ties to the lowest row:
// the candidate set and rule of LAPACK getrf), the pivot-row owners publish
// the normalised row, and every thread updates its tile with exactly one
// DFMA per entry (pivot row / pivot column zeroed first, the pivot row's
// multiplier is 1).  The arithmetic per entry does not depend on the tile
// mapping: factors are bitwise those of any other mapping.
template <int SZ>
__global__ void __launch_bounds__(GJShape<SZ>::THREADS, (GJShape<SZ>::THREADS <= 256 ? 2 : 1))
k_gj_inverse(const double* __restrict__ BT, double* __restrict__ XT, uint8_t* __restrict__ perm, Status* st,
             const int* __restrict__ in_slot, const int* __restrict__ out_idx, int bad_kind) {
  using S = GJShape<SZ>;
  constexpr int TR = S::TR, TC = S::TC, NRG = S::NRG, NCG = S::NCG, RPL = S::ROWS_PER_LANE;
  __shared__ double colbuf[2][SZ];
  __shared__ double rowbuf[2][SZ];
  __shared__ int pivs[SZ];
  __shared__ int s_bad;
  // optional gather / scatter: block in_slot[b] of BT -> factor out_idx[b]
  const int64_t e = out_idx ? (int64_t)out_idx[blockIdx.x] : (int64_t)blockIdx.x;
  const int64_t e_in = in_slot ? (int64_t)in_slot[blockIdx.x] : (int64_t)blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const bool active = tid < NRG * NCG;
  const int rg = tid % NRG, cg = tid / NRG;
  const int c0 = cg * TC;
  const double* src = BT + e_in * (int64_t)SZ * SZ;
  double a[TR][TC];
#pragma unroll
  for (int j = 0; j < TC; ++j) {
#pragma unroll
    for (int i = 0; i < TR; ++i) {
      const int r = rg + NRG * i, c = c0 + j;
      a[i][j] = (active && r < SZ && c < SZ) ? __ldg(src + (int64_t)c * SZ + r) : 0.0;
    }
  }
  if (tid == 0) s_bad = 0;
  unsigned used = 0;  // bit m: row lane + 32 m already pivoted (same in every warp)
  for (int kg = 0; kg < NCG; ++kg) {
#pragma unroll
    for (int kk = 0; kk < TC; ++kk) {
      const int k = kg * TC + kk;
      if (k >= SZ) break;
      double* cb = colbuf[k & 1];
      double* rb = rowbuf[k & 1];
      const bool colown = active && cg == kg;
      if (colown) {
#pragma unroll
        for (int i = 0; i < TR; ++i)
          if (rg + NRG * i < SZ) cb[rg + NRG * i] = a[i][kk];
      }
      __syncthreads();
      double best = -1.0;
      int brow = -1;
#pragma unroll
      for (int m = 0; m < RPL; ++m) {
        const int r = lane + 32 * m;
        if (r < SZ && !((used >> m) & 1u)) {
          const double v = fabs(cb[r]);
          if (v > best) {
            best = v;
            brow = r;
          }
        }
      }
      // warp arg-max, ties to the lowest row (rows of different lanes interleave)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int orow = __shfl_xor_sync(0xffffffffu, brow, off);
        if (orow >= 0 && (brow < 0 || ov > best || (ov == best && orow < brow))) {
          best = ov;
          brow = orow;
        }
      }
      const bool nan_col = brow < 0;
      const int p = nan_col ? k : brow;  // every candidate NaN: flagged singular below
      if (!nan_col && lane == (p & 31)) used |= 1u << (p >> 5);
      const double pv = cb[p];
      if (tid == 0) {
        pivs[k] = p;
        if (nan_col || !(pv != 0.0) || !isfinite(pv)) s_bad = 1;
      }
      const double pinv = 1.0 / pv;
      const bool rowown = active && rg == p % NRG;
      const int ip = p / NRG;
      if (rowown) {
#pragma unroll
        for (int i = 0; i < TR; ++i) {
          if (i == ip) {
#pragma unroll
            for (int j = 0; j < TC; ++j) {
              const int c = c0 + j;
              if (c < SZ) rb[c] = ((cg == kg && j == kk) ? 1.0 : a[i][j]) * pinv;
            }
          }
        }
      }
      __syncthreads();
      if (active) {
        double g[TR];
#pragma unroll
        for (int i = 0; i < TR; ++i) {
          const int r = rg + NRG * i;
          g[i] = (r < SZ) ? ((r == p) ? 1.0 : -cb[r]) : 0.0;
        }
        if (colown) {
#pragma unroll
          for (int i = 0; i < TR; ++i) a[i][kk] = 0.0;
        }
        if (rowown) {
#pragma unroll
          for (int i = 0; i < TR; ++i)
            if (i == ip) {
#pragma unroll
              for (int j = 0; j < TC; ++j) a[i][j] = 0.0;
            }
        }
        double pr[TC];
#pragma unroll
        for (int j = 0; j < TC; ++j) pr[j] = (c0 + j < SZ) ? rb[c0 + j] : 0.0;
#pragma unroll
        for (int i = 0; i < TR; ++i) {
#pragma unroll
          for (int j = 0; j < TC; ++j) a[i][j] = fma(g[i], pr[j], a[i][j]);
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0 && s_bad && st != nullptr) {
    if (atomicCAS(&st->kind, 0, bad_kind) == 0) st->element = e;
  }
  double* dst = XT + e * (int64_t)SZ * SZ;
  if (active) {
#pragma unroll
    for (int j = 0; j < TC; ++j) {
#pragma unroll
      for (int i = 0; i < TR; ++i) {
        const int r = rg + NRG * i, c = c0 + j;
        if (r < SZ && c < SZ) dst[(int64_t)c * SZ + r] = a[i][j];
      }
    }
  }
  uint8_t* pe = perm + e * 2 * SZ;
  for (int k = tid; k < SZ; k += blockDim.x) {
    const int p = pivs[k];
    pe[k] = (uint8_t)p;
    pe[SZ + p] = (uint8_t)k;
  }
}

// y[q_r] = sum_c XT[c][r] x[p_c]  (optionally out = base + omega * y, pmg.py:164)
// Thread per (element, r); the CTA stages the gathered x[p_c] of its
// elements in shared memory.
template <bool UPDATE>
__global__ void __launch_bounds__(256)
k_block_gemv(int64_t M, int SZ, const double* __restrict__ XT, const uint8_t* __restrict__ perm,
             const double* __restrict__ x, double omega, const double* __restrict__ base,
             double* __restrict__ out) {
  extern __shared__ double xs[];
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t total = M * SZ;
  const int64_t e_first = t0 / SZ;
  int64_t e_last = (t0 + blockDim.x - 1) / SZ;
  if (e_last > M - 1) e_last = M - 1;
  const int span = (int)(e_last - e_first + 1);
  for (int i = threadIdx.x; i < span * SZ; i += blockDim.x) {
    const int el = i / SZ, c = i - el * SZ;
    const int64_t e = e_first + el;
    const int pc = perm[e * 2 * SZ + c];
    xs[i] = __ldg(x + e * SZ + pc);
  }
  __syncthreads();
  const int64_t t = t0 + threadIdx.x;
  if (t >= total) return;
  const int64_t e = t / SZ;
  const int r = (int)(t - e * SZ);
  const double* Ae = XT + e * (int64_t)SZ * SZ + r;
  const double* xe = xs + (e - e_first) * SZ;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int c = 0;
  for (; c + 4 <= SZ; c += 4) {
    a0 += __ldg(Ae + (int64_t)(c + 0) * SZ) * xe[c + 0];
    a1 += __ldg(Ae + (int64_t)(c + 1) * SZ) * xe[c + 1];
    a2 += __ldg(Ae + (int64_t)(c + 2) * SZ) * xe[c + 2];
    a3 += __ldg(Ae + (int64_t)(c + 3) * SZ) * xe[c + 3];
  }
  for (; c < SZ; ++c) a0 += __ldg(Ae + (int64_t)c * SZ) * xe[c];
  const double y = (a0 + a1) + (a2 + a3);
  const int64_t o = e * SZ + perm[e * 2 * SZ + SZ + r];
  if (UPDATE) out[o] = base[o] + omega * y;
  else out[o] = y;
}

// Same map, two adjacent rows per thread with 16-byte loads (SZ even).
template <bool UPDATE>
__global__ void __launch_bounds__(256)
k_block_gemv2(int64_t M, int SZ, const double* __restrict__ XT, const uint8_t* __restrict__ perm,
              const double* __restrict__ x, double omega, const double* __restrict__ base,
              double* __restrict__ out) {
  extern __shared__ double xs[];
  const int H = SZ >> 1;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t total = M * H;
  const int64_t e_first = t0 / H;
  int64_t e_last = (t0 + blockDim.x - 1) / H;
  if (e_last > M - 1) e_last = M - 1;
  const int span = (int)(e_last - e_first + 1);
  for (int i = threadIdx.x; i < span * SZ; i += blockDim.x) {
    const int el = i / SZ, c = i - el * SZ;
    const int64_t e = e_first + el;
    xs[i] = __ldg(x + e * SZ + perm[e * 2 * SZ + c]);
  }
  __syncthreads();
  const int64_t t = t0 + threadIdx.x;
  if (t >= total) return;
  const int64_t e = t / H;
  const int r = 2 * (int)(t - e * H);
  const double2* Ae = reinterpret_cast<const double2*>(XT + e * (int64_t)SZ * SZ + r);
  const int ld = H;  // in double2 units
  const double* xe = xs + (e - e_first) * SZ;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  int c = 0;
  for (; c + 4 <= SZ; c += 4) {
    const double2 v0 = __ldg(Ae + (int64_t)(c + 0) * ld);
    const double2 v1 = __ldg(Ae + (int64_t)(c + 1) * ld);
    const double2 v2 = __ldg(Ae + (int64_t)(c + 2) * ld);
    const double2 v3 = __ldg(Ae + (int64_t)(c + 3) * ld);
    const double x0 = xe[c], x1 = xe[c + 1], x2 = xe[c + 2], x3 = xe[c + 3];
    a0 += v0.x * x0;
    b0 += v0.y * x0;
    a1 += v1.x * x1;
    b1 += v1.y * x1;
    a0 += v2.x * x2;
    b0 += v2.y * x2;
    a1 += v3.x * x3;
    b1 += v3.y * x3;
  }
  for (; c < SZ; ++c) {
    const double2 v = __ldg(Ae + (int64_t)c * ld);
    a0 += v.x * xe[c];
    b0 += v.y * xe[c];
  }
  const uint8_t* q = perm + e * 2 * SZ + SZ;
  const int64_t o0 = e * SZ + q[r], o1 = e * SZ + q[r + 1];
  const double y0 = a0 + a1, y1 = b0 + b1;
  if (UPDATE) {
    out[o0] = base[o0] + omega * y0;
    out[o1] = base[o1] + omega * y1;
  } else {
    out[o0] = y0;
    out[o1] = y1;
  }
}

// FP32-stored factor (pmg.block_precision = fp32: half the bytes of the
// dominant HBM stream of a pMG step), FP64 arithmetic: the same map, four
// adjacent rows per thread with 16-byte float4 loads (SZ % 4 == 0), or one
// row per thread otherwise.  Each product is formed in FP64 from the
// widened FP32 entry.
template <bool UPDATE, int U>
__global__ void __launch_bounds__(256)
k_block_gemv4f(int64_t M, int SZ, const float* __restrict__ XT, const uint8_t* __restrict__ perm,
               const double* __restrict__ x, double omega, const double* __restrict__ base,
               double* __restrict__ out) {
  extern __shared__ double xs[];
  const int Q = SZ >> 2;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t total = M * Q;
  const int64_t e_first = t0 / Q;
  int64_t e_last = (t0 + blockDim.x - 1) / Q;
  if (e_last > M - 1) e_last = M - 1;
  const int span = (int)(e_last - e_first + 1);
  const int64_t t = t0 + threadIdx.x;
  const bool live = t < total;
  const int64_t e = live ? t / Q : e_first;
  const int r = live ? 4 * (int)(t - e * Q) : 0;
  const float4* Ae = reinterpret_cast<const float4*>(XT + e * (int64_t)SZ * SZ + r);
  // software pipeline: the first U factor columns are in flight while the
  // CTA gathers x[p_c] into shared memory (the gather is a dependent
  // perm -> x load chain, the fixed cost of every CTA)
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = live ? __ldg(Ae + (int64_t)u * Q) : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = threadIdx.x; i < span * SZ; i += blockDim.x) {
    const int el = i / SZ, c = i - el * SZ;
    const int64_t ee = e_first + el;
    xs[i] = __ldg(x + ee * SZ + perm[ee * 2 * SZ + c]);
  }
  __syncthreads();
  if (!live) return;
  const double* xe = xs + (e - e_first) * SZ;
  double a[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  // SZ % 4 == 0 and U = 4: whole batches; the next batch loads while this
  // one is consumed
  for (int c = 0; c < SZ; c += U) {
    float4 w[U];
    const bool more = c + U < SZ;
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = more ? __ldg(Ae + (int64_t)(c + U + u) * Q) : v[u];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double xu = xe[c + u];
      a[u & 1][0] += (double)v[u].x * xu;
      a[u & 1][1] += (double)v[u].y * xu;
      a[u & 1][2] += (double)v[u].z * xu;
      a[u & 1][3] += (double)v[u].w * xu;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = w[u];
  }
  const uint8_t* q = perm + e * 2 * SZ + SZ;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double y = a[0][k] + a[1][k];
    const int64_t o = e * SZ + q[r + k];
    out[o] = UPDATE ? base[o] + omega * y : y;
  }
}

template <bool UPDATE>
__global__ void __launch_bounds__(256)
k_block_gemv1f(int64_t M, int SZ, const float* __restrict__ XT, const uint8_t* __restrict__ perm,
               const double* __restrict__ x, double omega, const double* __restrict__ base,
               double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * SZ) return;
  const int64_t e = t / SZ;
  const int r = (int)(t - e * SZ);
  const float* Ae = XT + e * (int64_t)SZ * SZ + r;
  const uint8_t* pe = perm + e * 2 * SZ;
  double a = 0.0;
  for (int c = 0; c < SZ; ++c) a += (double)__ldg(Ae + (int64_t)c * SZ) * __ldg(x + e * SZ + pe[c]);
  const int64_t o = e * SZ + pe[SZ + r];
  out[o] = UPDATE ? base[o] + omega * a : a;
}

__global__ void __launch_bounds__(256) k_demote(int64_t n, const double* __restrict__ src, float* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __double2float_rn(src[i]);
}

// Block-CSR matvec y_i = sum_k A_k x_{j_k} (SparseBlockMatrix.matvec,
// newton_krylov.py:243-251): thread per (row, component r); each block's
// product is summed first and then added to the row accumulator, in the
// row's column order, as the reference does.  Blocks column-major.
__global__ void __launch_bounds__(256)
k_sparse_matvec(int64_t n_rows, int SZ, const int* __restrict__ indptr, const int* __restrict__ indices,
                const double* __restrict__ blocks, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_rows * SZ) return;
  const int64_t i = t / SZ;
  const int r = (int)(t - i * SZ);
  double acc = 0.0;
  for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
    const double* A = blocks + (int64_t)k * SZ * SZ + r;
    const double* xj = x + (int64_t)indices[k] * SZ;
    double s = 0.0;
    for (int c = 0; c < SZ; ++c) s = fma(A[(int64_t)c * SZ], __ldg(xj + c), s);
    acc += s;
  }
  y[t] = acc;
}

int launch_sparse_matvec(int64_t n_rows, int SZ, const int* indptr, const int* indices, const double* blocks,
                         const double* x, double* y, cudaStream_t st) {
  const int64_t n = n_rows * SZ;
  if (n <= 0) return 0;
  k_sparse_matvec<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n_rows, SZ, indptr, indices, blocks, x, y);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Block ILU0 with zero fill (ilu0_factor / ilu0_apply, newton_krylov.py:
// 319-368), level-scheduled: the host groups rows into levels of the
// lower-neighbour DAG (factor, forward sweep) and of the upper-neighbour
// DAG (backward sweep); rows of one level are independent and each row
// does exactly the reference's sequence of block operations.  Blocks are
// column-major (B[c*SZ + r] = B[r][c]); the inverted pivot blocks are kept
// in Gauss-Jordan factor form (XT, perm): Dinv[t][c] = XT[q_c*SZ + p_t].

// acc[i][j] = sum_t A[r0+i][t] B[t][c0+j]   (t ascending)
template <int SZ, bool BPERM>
__device__ __forceinline__ void tile_gemm(const double* __restrict__ A, const double* __restrict__ B,
                                          const uint8_t* __restrict__ perm, int r0, int c0,
                                          double (&acc)[GJShape<SZ>::TR][GJShape<SZ>::TC]) {
  constexpr int TR = GJShape<SZ>::TR, TC = GJShape<SZ>::TC;
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j) acc[i][j] = 0.0;
  int qc[TC];
#pragma unroll
  for (int j = 0; j < TC; ++j) qc[j] = (c0 + j < SZ) ? (BPERM ? (int)perm[SZ + c0 + j] : c0 + j) : 0;
  for (int t = 0; t < SZ; ++t) {
    const int pt = BPERM ? (int)perm[t] : t;
    double a[TR], b[TC];
#pragma unroll
    for (int i = 0; i < TR; ++i) a[i] = (r0 + i < SZ) ? A[t * SZ + r0 + i] : 0.0;
#pragma unroll
    for (int j = 0; j < TC; ++j) b[j] = (c0 + j < SZ) ? B[qc[j] * SZ + pt] : 0.0;
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
}

// One CTA per row i of the level: for every lower entry k (column kk < i,
// ascending): F_k <- F_k Dinv_kk, then F_k2 -= F_k F_(kk,j) for the row's
// entries k2 with column j > kk present in row kk.
template <int SZ>
__global__ void __launch_bounds__(GJShape<SZ>::THREADS)
k_ilu_level(const int* __restrict__ rows, const int* __restrict__ indptr, const int* __restrict__ indices,
            double* __restrict__ F, const double* __restrict__ DX, const uint8_t* __restrict__ DP) {
  using S = GJShape<SZ>;
  constexpr int TR = S::TR, TC = S::TC, NRG = S::NRG;
  const int i = rows[blockIdx.x];
  const int tid = threadIdx.x;
  const bool active = tid < NRG * S::NCG;
  const int r0 = (tid % NRG) * TR, c0 = (tid / NRG) * TC;
  const int lo = indptr[i], hi = indptr[i + 1];
  constexpr int64_t BB = (int64_t)SZ * SZ;
  double acc[TR][TC];
  for (int k = lo; k < hi; ++k) {
    const int kk = indices[k];
    if (kk >= i) break;  // columns are sorted: the lower entries come first
    double* Fk = F + k * BB;
    if (active) tile_gemm<SZ, true>(Fk, DX + kk * BB, DP + (int64_t)kk * 2 * SZ, r0, c0, acc);
    __syncthreads();  // every read of F_k done before it is overwritten
    if (active) {
#pragma unroll
      for (int j = 0; j < TC; ++j)
#pragma unroll
        for (int ii = 0; ii < TR; ++ii)
          if (r0 + ii < SZ && c0 + j < SZ) Fk[(c0 + j) * SZ + r0 + ii] = acc[ii][j];
    }
    __syncthreads();
    const int klo = indptr[kk], khi = indptr[kk + 1];
    for (int k2 = lo; k2 < hi; ++k2) {
      const int j2 = indices[k2];
      if (j2 <= kk) continue;
      int u = -1;
      for (int t = klo; t < khi; ++t)
        if (indices[t] == j2) u = t;
      if (u < 0) continue;
      if (active) {
        tile_gemm<SZ, false>(Fk, F + u * BB, nullptr, r0, c0, acc);
        double* Fk2 = F + k2 * BB;
#pragma unroll
        for (int j = 0; j < TC; ++j)
#pragma unroll
          for (int ii = 0; ii < TR; ++ii)
            if (r0 + ii < SZ && c0 + j < SZ) {
              double* x = Fk2 + (c0 + j) * SZ + r0 + ii;
              *x = *x - acc[ii][j];
            }
      }
    }
    __syncthreads();  // row blocks final before the next lower entry reads them
  }
}

// Sweeps.  One CTA per row of the level; the row's CSR entries go to
// shared memory first so that every block-row product of the row is issued
// at once (compile-time SZ, entries bounded by MAXNZ): the chain of
// dependent global loads is what bounds these tiny kernels.
constexpr int ILU_MAXNZ = 9;  // diagonal + at most 4 face neighbours (+ headroom)

// sum_c A[c][r] v[c] (column-major A offset to row r), loads batched ahead
// of their FMAs (12 in flight) -- the FMA order stays c ascending
template <int SZ>
__device__ __forceinline__ double dot_col(const double* __restrict__ A, const double* v) {
  constexpr int CH = 12;
  double s = 0.0;
#pragma unroll
  for (int c0 = 0; c0 < SZ; c0 += CH) {
    double a[CH], b[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (c0 + u < SZ) {
        a[u] = __ldg(A + (c0 + u) * SZ);
        b[u] = v[c0 + u];
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u)
      if (c0 + u < SZ) s = fma(a[u], b[u], s);
  }
  return s;
}

template <int SZ, bool UPPER>
__device__ __forceinline__ double ilu_row_sum(int i, int r, const int* __restrict__ indptr,
                                              const int* __restrict__ indices, const double* __restrict__ F,
                                              const double* __restrict__ v, int* sk, int* sj, int& nsel,
                                              double base) {
  if (threadIdx.x == 0) {
    const int lo = indptr[i], hi = indptr[i + 1];
    int n = 0;
    for (int k = lo; k < hi && n < ILU_MAXNZ; ++k) {
      const int j = indices[k];
      if (UPPER ? (j > i) : (j < i)) {
        sk[n] = k;
        sj[n] = j;
        ++n;
      }
    }
    sk[ILU_MAXNZ] = n;
  }
  __syncthreads();
  nsel = sk[ILU_MAXNZ];
  constexpr int64_t BB = (int64_t)SZ * SZ;
  double part[ILU_MAXNZ];
#pragma unroll
  for (int e = 0; e < ILU_MAXNZ; ++e) {
    part[e] = 0.0;
    if (e < nsel && r < SZ) {
      part[e] = dot_col<SZ>(F + sk[e] * BB + r, v + (int64_t)sj[e] * SZ);
    }
  }
  // subtract in the row's column order, as acc -= block @ v_j does
  double acc = base;
#pragma unroll
  for (int e = 0; e < ILU_MAXNZ; ++e)
    if (e < nsel) acc -= part[e];
  return acc;
}

// forward sweep, unit lower factor: y_i = x_i - sum_{j<i} F_k y_j
template <int SZ>
__global__ void __launch_bounds__((SZ + 31) / 32 * 32)
k_ilu_forward(const int* __restrict__ rows, const int* __restrict__ indptr, const int* __restrict__ indices,
              const double* __restrict__ F, const double* __restrict__ x, double* __restrict__ y) {
  __shared__ int sk[ILU_MAXNZ + 1], sj[ILU_MAXNZ];
  const int i = rows[blockIdx.x];
  const int r = threadIdx.x;
  int nsel;
  const double xr = r < SZ ? x[(int64_t)i * SZ + r] : 0.0;
  const double acc = ilu_row_sum<SZ, false>(i, r, indptr, indices, F, y, sk, sj, nsel, xr);
  if (r < SZ) y[(int64_t)i * SZ + r] = acc;
}

// backward sweep: out_i = Dinv_i (y_i - sum_{j>i} F_k out_j)
template <int SZ>
__global__ void __launch_bounds__((SZ + 31) / 32 * 32)
k_ilu_backward(const int* __restrict__ rows, const int* __restrict__ indptr, const int* __restrict__ indices,
               const double* __restrict__ F, const double* __restrict__ DX, const uint8_t* __restrict__ DP,
               const double* __restrict__ y, double* __restrict__ out) {
  __shared__ int sk[ILU_MAXNZ + 1], sj[ILU_MAXNZ];
  __shared__ double sacc[SZ];
  __shared__ uint8_t sp[2 * SZ];
  const int i = rows[blockIdx.x];
  const int r = threadIdx.x;
  constexpr int64_t BB = (int64_t)SZ * SZ;
  for (int t = r; t < 2 * SZ; t += blockDim.x) sp[t] = DP[(int64_t)i * 2 * SZ + t];
  int nsel;
  const double yr = r < SZ ? y[(int64_t)i * SZ + r] : 0.0;
  const double acc = ilu_row_sum<SZ, true>(i, r, indptr, indices, F, out, sk, sj, nsel, yr);
  if (r < SZ) sacc[r] = acc;
  __syncthreads();
  if (r < SZ) {
    const double* XT = DX + (int64_t)i * BB + r;
    constexpr int CH = 12;
    double s = 0.0;
#pragma unroll
    for (int c0 = 0; c0 < SZ; c0 += CH) {
      double a[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (c0 + u < SZ) a[u] = __ldg(XT + (c0 + u) * SZ);
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (c0 + u < SZ) s = fma(a[u], sacc[sp[c0 + u]], s);
    }
    out[(int64_t)i * SZ + sp[SZ + r]] = s;
  }
}

// Persistent sweeps: one co-resident grid walks all forward levels, then
// all backward levels, with a global barrier between levels; each CTA
// takes rows b, b + G, ... of a level.  Same per-row arithmetic as the
// per-level kernels above.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// sense barrier over a co-resident grid: the generation is read (acquire,
// device scope -- a volatile load would be system scope and slow) before
// arriving; the last arriver resets the count and bumps the generation
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire_gpu(gen);
    __threadfence();  // this CTA's writes before the arrival
    if (atom_add_acq_rel_gpu(count, 1u) == nblocks - 1) {
      *count = 0;
      atom_add_acq_rel_gpu(gen, 1u);
    } else {
      while (ld_acquire_gpu(gen) == g) {
      }
    }
  }
  __syncthreads();
}

// dense per-row entry lists: ent[i*8 + e] = (slot, column) of the row's
// e-th lower (e < 4) / upper (4 <= e < 8) block in CSR order, -1 padded
constexpr int ILU_ENT = 4;

template <int SZ>
__device__ __forceinline__ double ilu_row_dense(int i, int r, const int2* __restrict__ ent, int half,
                                                const double* __restrict__ F, const double* __restrict__ v,
                                                double base) {
  constexpr int64_t BB = (int64_t)SZ * SZ;
  int2 en[ILU_ENT];
#pragma unroll
  for (int e = 0; e < ILU_ENT; ++e) en[e] = __ldg(ent + (int64_t)i * 2 * ILU_ENT + half * ILU_ENT + e);
  double part[ILU_ENT];
#pragma unroll
  for (int e = 0; e < ILU_ENT; ++e) {
    part[e] = 0.0;
    if (en[e].x >= 0 && r < SZ) part[e] = dot_col<SZ>(F + en[e].x * BB + r, v + (int64_t)en[e].y * SZ);
  }
  double acc = base;
#pragma unroll
  for (int e = 0; e < ILU_ENT; ++e)
    if (en[e].x >= 0) acc -= part[e];
  return acc;
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// prefetch into L2 the blocks of this CTA's rows in the next level
template <int SZ>
__device__ __forceinline__ void ilu_prefetch(const int* __restrict__ lptr, const int* __restrict__ lrows, int L1,
                                             int nlev, const int2* __restrict__ ent, int half,
                                             const double* __restrict__ F) {
  if (L1 >= nlev) return;
  constexpr int64_t BB = (int64_t)SZ * SZ;
  constexpr int LINES = (int)((BB * 8 + 127) / 128);
  for (int t = lptr[L1] + blockIdx.x; t < lptr[L1 + 1]; t += gridDim.x) {
    const int i = lrows[t];
#pragma unroll
    for (int e = 0; e < ILU_ENT; ++e) {
      const int2 en = __ldg(ent + (int64_t)i * 2 * ILU_ENT + half * ILU_ENT + e);
      if (en.x < 0) continue;
      const char* b = reinterpret_cast<const char*>(F + en.x * BB);
      for (int l = threadIdx.x; l < LINES; l += blockDim.x) prefetch_l2(b + l * 128);
    }
  }
}

template <int SZ>
__global__ void __launch_bounds__((SZ + 31) / 32 * 32)
k_ilu_apply_persistent(int n_lo, const int* __restrict__ lo_ptr, const int* __restrict__ lo_rows, int n_up,
                       const int* __restrict__ up_ptr, const int* __restrict__ up_rows,
                       const int2* __restrict__ ent, const double* __restrict__ F, const double* __restrict__ DX,
                       const uint8_t* __restrict__ DP, const double* __restrict__ x, double* __restrict__ y,
                       double* __restrict__ out, unsigned* bar) {
  __shared__ double sacc[SZ];
  __shared__ uint8_t sp[2 * SZ];
  const unsigned G = gridDim.x;
  const int r = threadIdx.x;
  constexpr int64_t BB = (int64_t)SZ * SZ;
  ilu_prefetch<SZ>(lo_ptr, lo_rows, 0, n_lo, ent, 0, F);
  for (int L = 0; L < n_lo; ++L) {
    for (int t = lo_ptr[L] + blockIdx.x; t < lo_ptr[L + 1]; t += G) {
      const int i = lo_rows[t];
      const double xr = r < SZ ? x[(int64_t)i * SZ + r] : 0.0;
      const double acc = ilu_row_dense<SZ>(i, r, ent, 0, F, y, xr);
      if (r < SZ) y[(int64_t)i * SZ + r] = acc;
    }
    ilu_prefetch<SZ>(lo_ptr, lo_rows, L + 1, n_lo, ent, 0, F);
    if (L + 1 == n_lo) ilu_prefetch<SZ>(up_ptr, up_rows, 0, n_up, ent, 1, F);
    grid_barrier(bar, bar + 1, G);
  }
  for (int L = 0; L < n_up; ++L) {
    for (int t = up_ptr[L] + blockIdx.x; t < up_ptr[L + 1]; t += G) {
      const int i = up_rows[t];
      for (int u = r; u < 2 * SZ; u += blockDim.x) sp[u] = DP[(int64_t)i * 2 * SZ + u];
      const double yr = r < SZ ? y[(int64_t)i * SZ + r] : 0.0;
      const double acc = ilu_row_dense<SZ>(i, r, ent, 1, F, out, yr);
      if (r < SZ) sacc[r] = acc;
      __syncthreads();
      if (r < SZ) {
        const double* XT = DX + (int64_t)i * BB + r;
        constexpr int CH = 12;
        double s = 0.0;
#pragma unroll
        for (int c0 = 0; c0 < SZ; c0 += CH) {
          double a[CH];
#pragma unroll
          for (int u = 0; u < CH; ++u)
            if (c0 + u < SZ) a[u] = __ldg(XT + (c0 + u) * SZ);
#pragma unroll
          for (int u = 0; u < CH; ++u)
            if (c0 + u < SZ) s = fma(a[u], sacc[sp[c0 + u]], s);
        }
        out[(int64_t)i * SZ + sp[SZ + r]] = s;
      }
      __syncthreads();
    }
    ilu_prefetch<SZ>(up_ptr, up_rows, L + 1, n_up, ent, 1, F);
    grid_barrier(bar, bar + 1, G);
  }
}

template <int SZ>
static int run_ilu_persistent(int n_lo, const int* lo_ptr, const int* lo_rows, int n_up, const int* up_ptr,
                              const int* up_rows, const int2* ent, const double* F,
                              const double* DX, const uint8_t* DP, const double* x, double* y, double* out,
                              unsigned* bar, int max_rows, cudaStream_t st) {
  constexpr int TH = (SZ + 31) / 32 * 32;
  static std::atomic<int> resident_of[64];  // co-resident CTAs, per device (0 = not yet known)
  int dev = 0;
  cudaGetDevice(&dev);
  int resident = resident_of[dev & 63].load();
  if (resident == 0) {  // idempotent: racing threads compute the same value
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ilu_apply_persistent<SZ>, TH, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident = per_sm * sms;
    resident_of[dev & 63].store(resident);
  }
  int grid = max_rows < resident ? max_rows : resident;
  if (grid < 1) grid = 1;
  cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st);
  void* args[] = {&n_lo, &lo_ptr, &lo_rows, &n_up, &up_ptr, &up_rows, &ent, &F, &DX, &DP, &x, &y, &out, &bar};
  cudaLaunchCooperativeKernel((void*)k_ilu_apply_persistent<SZ>, dim3(grid), dim3(TH), args, 0, st);
  return (int)cudaGetLastError();
}

int launch_ilu_persistent(int SZ, int n_lo, const int* lo_ptr, const int* lo_rows, int n_up, const int* up_ptr,
                          const int* up_rows, const int* ent, const double* F,
                          const double* DX, const uint8_t* DP, const double* x, double* y, double* out,
                          unsigned* bar, int max_rows, cudaStream_t st) {
  switch (SZ) {
#define PMGB_PS(Z) \
  case Z: return run_ilu_persistent<Z>(n_lo, lo_ptr, lo_rows, n_up, up_ptr, up_rows, \
                                       reinterpret_cast<const int2*>(ent), F, DX, DP, \
                                       x, y, out, bar, max_rows, st);
    PMGB_PS(1) PMGB_PS(4) PMGB_PS(9) PMGB_PS(16) PMGB_PS(25) PMGB_PS(36) PMGB_PS(64) PMGB_PS(100) PMGB_PS(144)
#undef PMGB_PS
  }
  return -1000;
}

template <int SZ>
static int run_ilu_level(int64_t n, const int* rows, const int* indptr, const int* indices, double* F,
                         const double* DX, const uint8_t* DP, cudaStream_t st) {
  k_ilu_level<SZ><<<(unsigned)n, GJShape<SZ>::THREADS, 0, st>>>(rows, indptr, indices, F, DX, DP);
  return (int)cudaGetLastError();
}

int launch_ilu_level(int64_t n, int SZ, const int* rows, const int* indptr, const int* indices, double* F,
                     const double* DX, const uint8_t* DP, cudaStream_t st) {
  if (n <= 0) return 0;
  switch (SZ) {
    case 1: return run_ilu_level<1>(n, rows, indptr, indices, F, DX, DP, st);
    case 4: return run_ilu_level<4>(n, rows, indptr, indices, F, DX, DP, st);
    case 9: return run_ilu_level<9>(n, rows, indptr, indices, F, DX, DP, st);
    case 16: return run_ilu_level<16>(n, rows, indptr, indices, F, DX, DP, st);
    case 25: return run_ilu_level<25>(n, rows, indptr, indices, F, DX, DP, st);
    case 36: return run_ilu_level<36>(n, rows, indptr, indices, F, DX, DP, st);
    case 64: return run_ilu_level<64>(n, rows, indptr, indices, F, DX, DP, st);
    case 100: return run_ilu_level<100>(n, rows, indptr, indices, F, DX, DP, st);
    case 144: return run_ilu_level<144>(n, rows, indptr, indices, F, DX, DP, st);
  }
  return -1000;
}

template <int SZ>
static int run_ilu_sweep(int backward, int64_t n, const int* rows, const int* indptr, const int* indices,
                         const double* F, const double* DX, const uint8_t* DP, const double* in, double* out,
                         cudaStream_t st) {
  constexpr int TH = (SZ + 31) / 32 * 32;
  if (backward)
    k_ilu_backward<SZ><<<(unsigned)n, TH, 0, st>>>(rows, indptr, indices, F, DX, DP, in, out);
  else
    k_ilu_forward<SZ><<<(unsigned)n, TH, 0, st>>>(rows, indptr, indices, F, in, out);
  return (int)cudaGetLastError();
}

int launch_ilu_sweep(int backward, int64_t n, int SZ, const int* rows, const int* indptr, const int* indices,
                     const double* F, const double* DX, const uint8_t* DP, const double* in, double* out,
                     cudaStream_t st) {
  if (n <= 0) return 0;
  switch (SZ) {
#define PMGB_SW(Z) case Z: return run_ilu_sweep<Z>(backward, n, rows, indptr, indices, F, DX, DP, in, out, st);
    PMGB_SW(1) PMGB_SW(4) PMGB_SW(9) PMGB_SW(16) PMGB_SW(25) PMGB_SW(36) PMGB_SW(64) PMGB_SW(100) PMGB_SW(144)
#undef PMGB_SW
  }
  return -1000;
}

template <int SZ>
static int run_gj(int64_t M, const double* BT, double* XT, uint8_t* perm, cudaStream_t st, Status* stp,
                  const int* in_slot, const int* out_idx, int bad_kind) {
  k_gj_inverse<SZ><<<(unsigned)M, GJShape<SZ>::THREADS, 0, st>>>(BT, XT, perm, stp, in_slot, out_idx, bad_kind);
  return (int)cudaGetLastError();
}

int launch_inverse(int64_t M, int SZ, const double* BT, double* XT, uint8_t* perm, cudaStream_t st,
                   Status* stp, const int* in_slot, const int* out_idx, int bad_kind) {
  if (M <= 0) return 0;
  switch (SZ) {
    case 1: return run_gj<1>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 4: return run_gj<4>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 9: return run_gj<9>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 16: return run_gj<16>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 25: return run_gj<25>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 36: return run_gj<36>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 64: return run_gj<64>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 100: return run_gj<100>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
    case 144: return run_gj<144>(M, BT, XT, perm, st, stp, in_slot, out_idx, bad_kind);
  }
  return -1000;
}

int launch_block_gemv(int64_t M, int SZ, const double* XT, const uint8_t* perm, const double* x, double omega,
                      const double* base, double* out, cudaStream_t st) {
  const int64_t n = M * SZ;
  if (n <= 0) return 0;
  if ((SZ & 1) == 0 && SZ >= 16) {
    const int64_t nt = M * (SZ / 2);
    const unsigned grid = (unsigned)((nt + 255) / 256);
    const size_t smem = sizeof(double) * (size_t)((255 / (SZ / 2)) + 2) * SZ;
    if (base)
      k_block_gemv2<true><<<grid, 256, smem, st>>>(M, SZ, XT, perm, x, omega, base, out);
    else
      k_block_gemv2<false><<<grid, 256, smem, st>>>(M, SZ, XT, perm, x, 0.0, nullptr, out);
    return (int)cudaGetLastError();
  }
  const unsigned grid = (unsigned)((n + 255) / 256);
  const size_t smem = sizeof(double) * (size_t)((255 / SZ) + 2) * SZ;
  if (base)
    k_block_gemv<true><<<grid, 256, smem, st>>>(M, SZ, XT, perm, x, omega, base, out);
  else
    k_block_gemv<false><<<grid, 256, smem, st>>>(M, SZ, XT, perm, x, 0.0, nullptr, out);
  return (int)cudaGetLastError();
}

int launch_block_gemv_f32(int64_t M, int SZ, const float* XT, const uint8_t* perm, const double* x, double omega,
                          const double* base, double* out, cudaStream_t st) {
  const int64_t n = M * SZ;
  if (n <= 0) return 0;
  if ((SZ & 3) == 0) {
    const int64_t nt = M * (SZ / 4);
    const unsigned grid = (unsigned)((nt + 255) / 256);
    const size_t smem = sizeof(double) * (size_t)((255 / (SZ / 4)) + 2) * SZ;
    if (base)
      k_block_gemv4f<true, 4><<<grid, 256, smem, st>>>(M, SZ, XT, perm, x, omega, base, out);
    else
      k_block_gemv4f<false, 4><<<grid, 256, smem, st>>>(M, SZ, XT, perm, x, 0.0, nullptr, out);
    return (int)cudaGetLastError();
  }
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (base)
    k_block_gemv1f<true><<<grid, 256, 0, st>>>(M, SZ, XT, perm, x, omega, base, out);
  else
    k_block_gemv1f<false><<<grid, 256, 0, st>>>(M, SZ, XT, perm, x, 0.0, nullptr, out);
  return (int)cudaGetLastError();
}

int launch_demote(int64_t n, const double* src, float* dst, cudaStream_t st) {
  if (n <= 0) return 0;
  k_demote<<<148 * 8, 256, 0, st>>>(n, src, dst);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// pMG transfers (pmg.py:117-136), per element and variable:
//   dst[a][b] (+)= sum_ij T[a][i] T[b][j] (src - src_base)[i][j]
// The CTA stages its elements' inputs in shared memory (coalesced), then
// contracts separably: tmp[i][b] = sum_j T[b][j] s[i][j]; out = sum_i T[a][i] tmp[i][b].

struct TransferOp {
  double T[36];  // (n_out x n_in) row-major
};

constexpr int TR_THREADS = 256;

__global__ void __launch_bounds__(TR_THREADS)
k_transfer(int64_t M, int nv, int nin, int nout, int epb, const TransferOp op, const double* __restrict__ src,
           const double* __restrict__ src_base, double* __restrict__ dst, int accumulate) {
  extern __shared__ double sm[];
  const int in_sz = nin * nin * nv, mid_sz = nin * nout * nv, out_sz = nout * nout * nv;
  double* s_in = sm;                       // epb * in_sz
  double* s_mid = sm + epb * in_sz;        // epb * mid_sz
  const int64_t e0 = (int64_t)blockIdx.x * epb;
  const int64_t ne = (M - e0) < epb ? (M - e0) : epb;
  const int64_t nin_vals = ne * in_sz;
  const double* sb = src + e0 * in_sz;
  const double* bb = src_base ? src_base + e0 * in_sz : nullptr;
  for (int i = threadIdx.x; i < nin_vals; i += blockDim.x) {
    double v = __ldg(sb + i);
    if (bb) v = v - __ldg(bb + i);
    s_in[i] = v;
  }
  __syncthreads();
  // tmp[el][i][b][v] = sum_j T[b][j] s[el][i][j][v]
  for (int t = threadIdx.x; t < ne * mid_sz; t += blockDim.x) {
    const int el = t / mid_sz, r = t - el * mid_sz;
    const int v = r % nv, ib = r / nv, i = ib / nout, b = ib % nout;
    const double* s = s_in + el * in_sz + i * nin * nv + v;
    double acc = 0.0;
    for (int j = 0; j < nin; ++j) acc += op.T[b * nin + j] * s[j * nv];
    s_mid[t] = acc;
  }
  __syncthreads();
  double* db = dst + e0 * out_sz;
  for (int t = threadIdx.x; t < ne * out_sz; t += blockDim.x) {
    const int el = t / out_sz, r = t - el * out_sz;
    const int v = r % nv, ab = r / nv, a = ab / nout, b = ab % nout;
    const double* m = s_mid + el * mid_sz + b * nv + v;
    double acc = 0.0;
    for (int i = 0; i < nin; ++i) acc += op.T[a * nin + i] * m[i * nout * nv];
    if (accumulate) db[t] = db[t] + acc;
    else db[t] = acc;
  }
}

// Compile-time sizes for the flow kinds' level pairs (nv = 4): the same
// contractions in the same order as k_transfer (bitwise equal), without
// runtime divisions / loop bounds.  One CTA of 256 threads per EPB elements.
template <int NIN, int NOUT, int NV>
__global__ void __launch_bounds__(TR_THREADS)
k_transfer_t(int64_t M, const TransferOp op, const double* __restrict__ src, const double* __restrict__ src_base,
             double* __restrict__ dst, int accumulate) {
  constexpr int IN = NIN * NIN * NV, MID = NIN * NOUT * NV, OUT = NOUT * NOUT * NV;
  constexpr int EPB = (1024 / IN) < 1 ? 1 : ((1024 / IN) > 256 ? 256 : 1024 / IN);
  __shared__ double s_in[EPB * IN];
  __shared__ double s_mid[EPB * MID];
  const int64_t e0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((M - e0) < EPB ? (M - e0) : EPB);
  const double* sb = src + e0 * IN;
  const double* bb = src_base ? src_base + e0 * IN : nullptr;
  for (int i = threadIdx.x; i < ne * IN; i += TR_THREADS) {
    double v = __ldg(sb + i);
    if (bb) v = v - __ldg(bb + i);
    s_in[i] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ne * MID; t += TR_THREADS) {
    const int el = t / MID, r = t - el * MID;
    const int v = r % NV, ib = r / NV, i = ib / NOUT, b = ib % NOUT;
    const double* s = s_in + el * IN + i * NIN * NV + v;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < NIN; ++j) acc += op.T[b * NIN + j] * s[j * NV];
    s_mid[t] = acc;
  }
  __syncthreads();
  double* db = dst + e0 * OUT;
  for (int t = threadIdx.x; t < ne * OUT; t += TR_THREADS) {
    const int el = t / OUT, r = t - el * OUT;
    const int v = r % NV, ab = r / NV, a = ab / NOUT, b = ab % NOUT;
    const double* mm = s_mid + el * MID + b * NV + v;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < NIN; ++i) acc += op.T[a * NIN + i] * mm[i * NOUT * NV];
    if (accumulate) db[t] = db[t] + acc;
    else db[t] = acc;
  }
}

template <int NIN, int NOUT>
static int run_transfer_t(int64_t M, const TransferOp& op, const double* src, const double* src_base, double* dst,
                          int accumulate, cudaStream_t st) {
  constexpr int IN = NIN * NIN * 4;
  constexpr int EPB = (1024 / IN) < 1 ? 1 : ((1024 / IN) > 256 ? 256 : 1024 / IN);
  const unsigned grid = (unsigned)((M + EPB - 1) / EPB);
  k_transfer_t<NIN, NOUT, 4><<<grid, TR_THREADS, 0, st>>>(M, op, src, src_base, dst, accumulate);
  return (int)cudaGetLastError();
}

int launch_transfer(int64_t M, int nv, int nin, int nout, const double* T, const double* src,
                    const double* src_base, double* dst, int accumulate, cudaStream_t st) {
  TransferOp op;
  for (int i = 0; i < 36; ++i) op.T[i] = (i < nin * nout) ? T[i] : 0.0;
  if (M <= 0) return 0;
  static const bool generic = std::getenv("PMGB_TRANSFER_GENERIC") != nullptr;  // A/B only
  if (nv == 4 && !generic) {
    switch (nin * 8 + nout) {
#define PMGB_TR(A, B) case A * 8 + B: return run_transfer_t<A, B>(M, op, src, src_base, dst, accumulate, st);
      PMGB_TR(6, 5) PMGB_TR(5, 6) PMGB_TR(5, 4) PMGB_TR(4, 5) PMGB_TR(5, 3) PMGB_TR(3, 5) PMGB_TR(4, 3)
      PMGB_TR(3, 4) PMGB_TR(3, 2) PMGB_TR(2, 3) PMGB_TR(2, 1) PMGB_TR(1, 2) PMGB_TR(4, 2) PMGB_TR(2, 4)
#undef PMGB_TR
      default: break;
    }
  }
  const int in_sz = nin * nin * nv, mid_sz = nin * nout * nv;
  int epb = 1024 / (in_sz > 1 ? in_sz : 1);
  if (epb < 1) epb = 1;
  if (epb > 256) epb = 256;
  const size_t smem = sizeof(double) * (size_t)epb * (in_sz + mid_sz);
  const unsigned grid = (unsigned)((M + epb - 1) / epb);
  k_transfer<<<grid, TR_THREADS, smem, st>>>(M, nv, nin, nout, epb, op, src, src_base, dst, accumulate);
  return (int)cudaGetLastError();
}

}  // namespace pmgb
