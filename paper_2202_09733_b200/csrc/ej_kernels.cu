// Element-Jacobi blocks: batched in-place Gauss-Jordan inverse and the
// HBM-bound batched block GEMV / fused EJ sweep update.
//
// Reference: newton_krylov.py:187-210 (np.linalg.inv of the FD blocks,
// RuntimeError on a singular block), :157-171 (BlockJacobian.apply =
// einsum("mij,mj->mi")), pmg.py:162-164 (q <- q + omega B^-1 d).
//
// Storage: blocks and inverses are column-major per element (B^T
// row-major), so the GEMV thread for row i streams invT[e][j][i] with
// consecutive i across the warp (coalesced), x[e][j] is a broadcast.
#include <climits>

#include "pmgb_internal.cuh"

namespace pmgb {

// Gauss-Jordan with implicit partial pivoting (no row swaps): pivot of
// column k = largest |A[r][k]| over rows not yet used (ties -> lowest r),
// i.e. the same candidate set LAPACK's getrf searches after its swaps.
// Runs on A = B^T; the result is A^-1 = (B^-1)^T = invT, un-permuted on
// the store: A^-1[i][j] = X[prow[i]][q[j]], q = prow^-1.
__global__ void __launch_bounds__(256)
k_inverse(int SZ, const double* __restrict__ BT, double* __restrict__ invT, Status* st) {
  extern __shared__ double sm[];
  double* A = sm;                       // SZ*SZ
  double* col = A + SZ * SZ;            // SZ
  int* used = (int*)(col + SZ);         // SZ
  int* prow = used + SZ;                // SZ
  int* qinv = prow + SZ;                // SZ
  __shared__ int s_p;
  __shared__ double s_pv;
  __shared__ int s_bad;
  const int64_t e = blockIdx.x;
  const int tid = threadIdx.x, T = blockDim.x;
  const double* src = BT + e * (int64_t)SZ * SZ;
  for (int i = tid; i < SZ * SZ; i += T) A[i] = __ldg(src + i);
  for (int i = tid; i < SZ; i += T) used[i] = 0;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int k = 0; k < SZ; ++k) {
    if (tid < 32) {
      double bv = -1.0;
      int br = INT_MAX;
      for (int r = tid; r < SZ; r += 32) {
        if (!used[r]) {
          const double v = fabs(A[r * SZ + k]);
          if (v > bv || (v != v && bv == -1.0)) { bv = v; br = r; }
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, bv, off);
        const int orr = __shfl_down_sync(0xffffffffu, br, off);
        if (ov > bv || (ov == bv && orr < br)) { bv = ov; br = orr; }
      }
      if (tid == 0) {
        if (br == INT_MAX) br = k;  // all NaN: keep going, flagged below
        s_p = br;
        s_pv = A[br * SZ + k];
        used[br] = 1;
        prow[k] = br;
        qinv[br] = k;
        if (!(s_pv != 0.0) || !isfinite(s_pv)) s_bad = 1;
      }
    }
    __syncthreads();
    const int p = s_p;
    const double pinv = 1.0 / s_pv;
    for (int r = tid; r < SZ; r += T) col[r] = A[r * SZ + k];
    __syncthreads();
    for (int c = tid; c < SZ; c += T) A[p * SZ + c] = (c == k ? 1.0 : A[p * SZ + c]) * pinv;
    __syncthreads();
    for (int i = tid; i < SZ * SZ; i += T) {
      const int r = i / SZ, c = i - r * SZ;
      if (r == p) continue;
      const double a = (c == k) ? 0.0 : A[i];
      A[i] = a - col[r] * A[p * SZ + c];
    }
    __syncthreads();
  }
  if (tid == 0 && s_bad && st != nullptr) {
    if (atomicCAS(&st->kind, 0, 3) == 0) st->element = e;
  }
  double* dst = invT + e * (int64_t)SZ * SZ;
  for (int i = tid; i < SZ * SZ; i += T) {
    const int r = i / SZ, c = i - r * SZ;
    dst[i] = A[prow[r] * SZ + qinv[c]];
  }
}

// y[e][i] = sum_j invT[e][j][i] x[e][j]; optional fused EJ update
// out = base + omega * y   (pmg.py:164)
template <bool UPDATE>
__global__ void __launch_bounds__(256)
k_block_gemv(int64_t M, int SZ, const double* __restrict__ invT, const double* __restrict__ x,
             double omega, const double* __restrict__ base, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * SZ) return;
  const int64_t e = t / SZ;
  const int i = (int)(t - e * SZ);
  const double* Ae = invT + e * (int64_t)SZ * SZ + i;
  const double* xe = x + e * SZ;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = 0;
  for (; j + 4 <= SZ; j += 4) {
    a0 += __ldg(Ae + (int64_t)(j + 0) * SZ) * __ldg(xe + j + 0);
    a1 += __ldg(Ae + (int64_t)(j + 1) * SZ) * __ldg(xe + j + 1);
    a2 += __ldg(Ae + (int64_t)(j + 2) * SZ) * __ldg(xe + j + 2);
    a3 += __ldg(Ae + (int64_t)(j + 3) * SZ) * __ldg(xe + j + 3);
  }
  for (; j < SZ; ++j) a0 += __ldg(Ae + (int64_t)j * SZ) * __ldg(xe + j);
  const double y = (a0 + a1) + (a2 + a3);
  if (UPDATE) out[t] = base[t] + omega * y;
  else out[t] = y;
}

int launch_inverse(int64_t M, int SZ, const double* BT, double* invT, cudaStream_t st, Status* stp) {
  if (M <= 0) return 0;
  const size_t bytes = sizeof(double) * ((size_t)SZ * SZ + SZ) + sizeof(int) * 3 * SZ;
  static size_t attr = 0;
  if (bytes > attr) {
    cudaFuncSetAttribute(k_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr = bytes;
  }
  k_inverse<<<(unsigned)M, 256, bytes, st>>>(SZ, BT, invT, stp);
  return (int)cudaGetLastError();
}

int launch_block_gemv(int64_t M, int SZ, const double* invT, const double* x, double omega,
                      const double* base, double* out, cudaStream_t st) {
  const int64_t n = M * SZ;
  if (n <= 0) return 0;
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (base) k_block_gemv<true><<<grid, 256, 0, st>>>(M, SZ, invT, x, omega, base, out);
  else k_block_gemv<false><<<grid, 256, 0, st>>>(M, SZ, invT, x, 0.0, nullptr, out);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// pMG transfers (pmg.py:117-136): per element and variable
//   restrict: lo[a][b] = sum_ij G[a][i] G[b][j] hi[i][j]
//   prolong : hi[a][b] += sum_ij P[a][i] P[b][j] (lo - lo_base)[i][j]

struct TransferOp {
  double T[36];  // (n_out x n_in) row-major
};

__global__ void __launch_bounds__(256)
k_restrict(int64_t M, int nv, int nin, int nout, const TransferOp op, const double* __restrict__ src,
           const double* __restrict__ src_base, double* __restrict__ dst, int accumulate) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = nout * nout * nv;
  if (t >= M * per) return;
  const int64_t e = t / per;
  const int r = (int)(t - e * per);
  const int v = r % nv, pt = r / nv, a = pt / nout, b = pt % nout;
  const double* s = src + e * (int64_t)nin * nin * nv + v;
  const double* sb = src_base ? src_base + e * (int64_t)nin * nin * nv + v : nullptr;
  double acc = 0.0;
  for (int i = 0; i < nin; ++i) {
    const double ta = op.T[a * nin + i];
    for (int j = 0; j < nin; ++j) {
      double x = __ldg(s + (i * nin + j) * nv);
      if (sb) x = x - __ldg(sb + (i * nin + j) * nv);
      acc += (ta * op.T[b * nin + j]) * x;
    }
  }
  if (accumulate) dst[t] = dst[t] + acc;
  else dst[t] = acc;
}

int launch_transfer(int64_t M, int nv, int nin, int nout, const double* T, const double* src,
                    const double* src_base, double* dst, int accumulate, cudaStream_t st) {
  TransferOp op;
  for (int i = 0; i < 36; ++i) op.T[i] = (i < nin * nout) ? T[i] : 0.0;
  const int64_t n = M * nout * nout * nv;
  if (n <= 0) return 0;
  k_restrict<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(M, nv, nin, nout, op, src, src_base, dst, accumulate);
  return (int)cudaGetLastError();
}

}  // namespace pmgb
