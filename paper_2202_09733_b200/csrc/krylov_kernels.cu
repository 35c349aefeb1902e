// Deterministic BLAS-1 and Arnoldi (modified Gram-Schmidt) kernels.
//
// Reference: newton_krylov.py:79-151 (gmres_solve): H[i,j] = V_i . w,
// w -= H[i,j] V_i (:119-121), H[j+1,j] = ||w|| (:122), V_{j+1} = w/H
// (:124-127), x += P(V^T y) (:147-148); np.all(np.isfinite(w)) (:116).
//
// Every reduction uses a fixed grid, a fixed per-thread stride order, a
// fixed warp-shuffle tree and a fixed-order final pass by the last CTA
// to arrive (the arrival order never changes the arithmetic), so results
// are bitwise reproducible run to run -- the reference's residual logs
// are bitwise deterministic (tests/test_acceptance.py:472-501).
#include <cstdlib>
#include <map>
#include <mutex>

#include "pmgb_internal.cuh"

namespace pmgb {

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 148 * 8;  // fixed grid: reductions are order-deterministic

struct RedScratch {
  double* partial;          // RED_BLOCKS
  unsigned int* counter;    // 1
  int* flag;                // 1
};

// One scratch per (device, stream): a reduction's partials, its arrival
// counter and the finite flag are only ever touched by work queued on one
// stream, so reductions on different streams or devices never share them
// (reductions on one stream are ordered by the stream itself).
struct RedKey {
  int dev;
  cudaStream_t st;
  bool operator<(const RedKey& o) const { return dev != o.dev ? dev < o.dev : st < o.st; }
};
static std::mutex g_red_mu;
static std::map<RedKey, RedScratch> g_red;

static int red_scratch(RedScratch* out, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  std::lock_guard<std::mutex> lock(g_red_mu);
  auto it = g_red.find(RedKey{dev, st});
  if (it == g_red.end()) {
    void* p = nullptr;
    e = cudaMalloc(&p, sizeof(double) * RED_BLOCKS + 64);
    if (e != cudaSuccess) return (int)e;
    e = cudaMemset(p, 0, sizeof(double) * RED_BLOCKS + 64);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any stream uses it
    if (e != cudaSuccess) return (int)e;
    RedScratch rs;
    rs.partial = (double*)p;
    rs.counter = (unsigned int*)((char*)p + sizeof(double) * RED_BLOCKS);
    rs.flag = (int*)((char*)p + sizeof(double) * RED_BLOCKS + 16);
    it = g_red.emplace(RedKey{dev, st}, rs).first;
  }
  *out = it->second;
  return 0;
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[RED_THREADS / 32];
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (lane < RED_THREADS / 32) ? ws[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  }
  return s;  // valid in thread 0
}

// last-arriving CTA sums the partials in a fixed order
__device__ __forceinline__ bool finish(const RedScratch& rs, double mine, double* out, bool do_sqrt) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    rs.partial[blockIdx.x] = mine;
    __threadfence();
    const unsigned prev = atomicAdd(rs.counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += ((volatile double*)rs.partial)[i];
  v = block_sum(v);
  if (threadIdx.x == 0) {
    *out = do_sqrt ? sqrt(v) : v;
    *rs.counter = 0u;
  }
  return true;
}

// w <- w - h_prev * Vprev (if Vprev); out = Vnext . w  (Vnext may be w)
// optionally flags a non-finite w on the first pass.  Each thread walks
// a fixed sequence of 4-element chunks; all loads of a chunk are issued
// before any store (w and Vnext may alias), keeping 4 loads per stream
// in flight.
constexpr int CH = 4;

// L2 policy across the j+1 passes of one Arnoldi step: w (read and
// written by every pass) is loaded / stored with an evict_last policy and
// the Krylov vectors V_i with evict_first.  Same arithmetic (bitwise);
// measured 4 % faster per GMRES(30) cycle at config 2 (19.97 -> 19.22 ms,
// tools/time_mgs.py) -- not the 2x that a fully L2-resident w would give:
// a persisting-L2 set-aside of 40-100 MB changed nothing, so w does not
// stay resident against the 2x52 MB V stream.
#ifndef PMGB_MGS_L2_HINTS
#define PMGB_MGS_L2_HINTS 1
#endif
__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_hint(const double* a, unsigned long long pol) {
#if PMGB_MGS_L2_HINTS
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol) : "memory");
  return v;
#else
  return *a;
#endif
}
__device__ __forceinline__ void st_hint(double* a, double v, unsigned long long pol) {
#if PMGB_MGS_L2_HINTS
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
#else
  *a = v;
#endif
}

__global__ void __launch_bounds__(RED_THREADS)
k_mgs_pass(int64_t n, double* w, const double* __restrict__ Vprev, const double* hprev, const double* Vnext,
           double* out, int do_sqrt, int check_finite, RedScratch rs) {
  const double h = Vprev ? *hprev : 0.0;
  const unsigned long long keep = pol_evict_last(), stream = pol_evict_first();
  const unsigned long long pnext = (Vnext == w) ? keep : stream;
  double acc = 0.0;
  int bad = 0;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nchunks = n / CH;
  for (int64_t c = tid; c < nchunks; c += nthreads) {
    const int64_t i = c * CH;
    double wv[CH], vn[CH], vp[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) wv[u] = ld_hint(w + i + u, keep);
#pragma unroll
    for (int u = 0; u < CH; ++u) vn[u] = ld_hint(Vnext + i + u, pnext);
    if (Vprev) {
#pragma unroll
      for (int u = 0; u < CH; ++u) vp[u] = ld_hint(Vprev + i + u, stream);
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      double wi = wv[u];
      if (Vprev) wi = wi - h * vp[u];
      if (check_finite && !isfinite(wi)) bad = 1;
      if (Vnext == w) vn[u] = wi;
      acc += vn[u] * wi;
      wv[u] = wi;
    }
    if (Vprev) {
#pragma unroll
      for (int u = 0; u < CH; ++u) st_hint(w + i + u, wv[u], keep);
    }
  }
  for (int64_t i = nchunks * CH + tid; i < n; i += nthreads) {  // tail
    double wi = w[i];
    if (Vprev) {
      wi = wi - h * Vprev[i];
      w[i] = wi;
    }
    if (check_finite && !isfinite(wi)) bad = 1;
    acc += (Vnext == w ? wi : Vnext[i]) * wi;
  }
  if (check_finite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(rs.flag, 1);
  const double s = block_sum(acc);
  finish(rs, s, out, do_sqrt != 0);
}

__global__ void __launch_bounds__(RED_THREADS)
k_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ y, double* out, int do_sqrt,
      RedScratch rs) {
  double acc = 0.0;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nchunks = n / CH;
  for (int64_t c = tid; c < nchunks; c += nthreads) {
    const int64_t i = c * CH;
    double a[CH], b[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      a[u] = x[i + u];
      b[u] = y[i + u];
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) acc += a[u] * b[u];
  }
  for (int64_t i = nchunks * CH + tid; i < n; i += nthreads) acc += x[i] * y[i];
  const double s = block_sum(acc);
  finish(rs, s, out, do_sqrt != 0);
}

// V_{j+1} = w / H if H > thresh (newton_krylov.py:123-127)
__global__ void k_normalize(int64_t n, const double* __restrict__ w, const double* h, double thresh,
                            double* __restrict__ v) {
  const double hv = *h;
  if (!(hv > thresh)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) v[i] = w[i] / hv;
}

// out = sum_{i<k} c_i x_i  (coefficients by value, k <= 8)
struct Lin {
  double c[8];
  const double* x[8];
  int k;
};

__global__ void k_lincomb(int64_t n, const Lin L, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = L.c[0] * L.x[0][i];
    for (int j = 1; j < L.k; ++j) s = s + L.c[j] * L.x[j][i];
    out[i] = s;
  }
}

// out = V^T y with y on the device (x += P(V[:j].T @ y))
// (y staged in dynamic shared memory: any Krylov dimension up to
// GEMV_T_MAX_K, same summation order for every k)
constexpr int GEMV_T_MAX_K = 227 * 1024 / 8 - 64;
__global__ void k_gemv_t(int64_t n, int k, const double* __restrict__ V, int64_t ld, const double* y,
                         double* __restrict__ out) {
  extern __shared__ double ys[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += V[(int64_t)j * ld + i] * ys[j];
    out[i] = s;
  }
}

__global__ void k_any_nonzero(int64_t n, const double* __restrict__ x, int* flag) {
  int hit = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (x[i] != 0.0) hit = 1;
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicOr(flag, 1);
}

static unsigned ew_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

int launch_dot(int64_t n, const double* x, const double* y, double* out, int do_sqrt, cudaStream_t st) {
  RedScratch rs;
  int e = red_scratch(&rs, st);
  if (e) return e;
  k_dot<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, x, y, out, do_sqrt, rs);
  return (int)cudaGetLastError();
}

// One full MGS orthogonalisation of w against V[0..j] (row stride ld):
// H[0..j] and H[j+1] = ||w||, V[j+1] = w / H[j+1] when H[j+1] > thresh.
// The finite flag covers w as it enters (before any projection).
int launch_mgs(int64_t n, double* V, int64_t ld, int j, double* w, double* H, double thresh, int* finite_flag,
               cudaStream_t st) {
  RedScratch rs;
  int e = red_scratch(&rs, st);
  if (e) return e;
  cudaMemsetAsync(rs.flag, 0, sizeof(int), st);
  for (int i = 0; i <= j; ++i) {
    const double* Vprev = (i == 0) ? nullptr : V + (int64_t)(i - 1) * ld;
    const double* hprev = (i == 0) ? nullptr : H + (i - 1);
    k_mgs_pass<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, w, Vprev, hprev, V + (int64_t)i * ld, H + i, 0,
                                                   i == 0 ? 1 : 0, rs);
  }
  k_mgs_pass<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, w, V + (int64_t)j * ld, H + j, w, H + j + 1, 1, 0, rs);
  k_normalize<<<ew_grid(n), 256, 0, st>>>(n, w, H + j + 1, thresh, V + (int64_t)(j + 1) * ld);
  if (finite_flag) cudaMemcpyAsync(finite_flag, rs.flag, sizeof(int), cudaMemcpyDeviceToDevice, st);
  return (int)cudaGetLastError();
}

// One MGS pass on its own (the partitioned Arnoldi step all-reduces each
// partial dot between passes): w -= (*hprev) Vprev (Vprev may be NULL),
// then *out = Vnext . w over these n entries; first = 1 clears the finite
// flag and checks w as it enters.
int launch_mgs_pass(int64_t n, double* w, const double* Vprev, const double* hprev, const double* Vnext,
                    double* out, int first, int* finite_flag, cudaStream_t st) {
  RedScratch rs;
  int e = red_scratch(&rs, st);
  if (e) return e;
  if (first) cudaMemsetAsync(rs.flag, 0, sizeof(int), st);
  k_mgs_pass<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, w, Vprev, hprev, Vnext, out, 0, first, rs);
  if (finite_flag) cudaMemcpyAsync(finite_flag, rs.flag, sizeof(int), cudaMemcpyDeviceToDevice, st);
  return (int)cudaGetLastError();
}

__global__ void k_sqrt1(double* h) { *h = sqrt(*h); }

// *h = sqrt(*h) (the all-reduced w . w), then V_{j+1} = w / *h if > thresh
int launch_normalize_sqrt(int64_t n, const double* w, double* h, double thresh, double* v, cudaStream_t st) {
  k_sqrt1<<<1, 1, 0, st>>>(h);
  k_normalize<<<ew_grid(n), 256, 0, st>>>(n, w, h, thresh, v);
  return (int)cudaGetLastError();
}

int launch_lincomb(int64_t n, int k, const double* c, const double* const* xs, double* out, cudaStream_t st) {
  if (k < 1 || k > 8) return -1001;
  Lin L;
  for (int i = 0; i < 8; ++i) {
    L.c[i] = i < k ? c[i] : 0.0;
    L.x[i] = i < k ? xs[i] : nullptr;
  }
  L.k = k;
  k_lincomb<<<ew_grid(n), 256, 0, st>>>(n, L, out);
  return (int)cudaGetLastError();
}

// RK smoother local pseudo-time steps: dtau[e] = cfl / (s + lam[e])
// (IEEE division, rounded as the oracle's NumPy expression)
__global__ void k_rk_dtau(int64_t M, const double* __restrict__ lam, double s, double cfl,
                          double* __restrict__ dtau) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < M; e += (int64_t)gridDim.x * blockDim.x)
    dtau[e] = __ddiv_rn(cfl, __dadd_rn(s, lam[e]));
}

int launch_rk_dtau(int64_t M, const double* lam, double s, double cfl, double* dtau, cudaStream_t st) {
  if (M == 0) return 0;
  k_rk_dtau<<<ew_grid(M), 256, 0, st>>>(M, lam, s, cfl, dtau);
  return (int)cudaGetLastError();
}

int launch_gemv_t(int64_t n, int k, const double* V, int64_t ld, const double* y, double* out, cudaStream_t st) {
  if (k < 1 || k > GEMV_T_MAX_K) return -1001;
  const size_t smem = sizeof(double) * (size_t)k;
  if (smem > 48 * 1024) {
    static std::atomic<unsigned long long> seen{0};
    once_per_device(seen, [&] {
      cudaFuncSetAttribute(k_gemv_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * GEMV_T_MAX_K));
    });
  }
  k_gemv_t<<<ew_grid(n), 256, smem, st>>>(n, k, V, ld, y, out);
  return (int)cudaGetLastError();
}

int launch_any_nonzero(int64_t n, const double* x, int* flag_dev, cudaStream_t st) {
  cudaMemsetAsync(flag_dev, 0, sizeof(int), st);
  k_any_nonzero<<<ew_grid(n), 256, 0, st>>>(n, x, flag_dev);
  return (int)cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Classical Gram-Schmidt with reorthogonalisation (CGS2, option
// gmres.ortho = cgs2): one multi-dot per pass, so a partitioned Arnoldi
// step needs 3 all-reduces instead of the MGS order's j + 2.

constexpr int MD_BLOCKS = 148 * 4, MD_THREADS = 256, MD_CH = 8, MD_KMAX = 256;

struct MdScratch {
  double* partial;     // MD_BLOCKS * MD_KMAX
  unsigned int* counter;
};
static std::map<RedKey, MdScratch> g_md;

static int md_scratch(MdScratch* out, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  std::lock_guard<std::mutex> lock(g_red_mu);
  auto it = g_md.find(RedKey{dev, st});
  if (it == g_md.end()) {
    void* p = nullptr;
    const size_t bytes = sizeof(double) * MD_BLOCKS * MD_KMAX + 64;
    e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return (int)e;
    MdScratch ms;
    ms.partial = (double*)p;
    ms.counter = (unsigned int*)((char*)p + sizeof(double) * MD_BLOCKS * MD_KMAX);
    it = g_md.emplace(RedKey{dev, st}, ms).first;
  }
  *out = it->second;
  return 0;
}

// block-wide sum of one value per thread, valid in thread 0; safe to call
// back to back (trailing barrier)
__device__ __forceinline__ double block_sum_md(double v, double* ws) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (lane < MD_THREADS / 32) ? ws[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  }
  __syncthreads();
  return s;
}

// out[c] = V_c . w for c < k (fixed grid, fixed per-thread order, fixed
// trees, last block sums the partials in block order: deterministic);
// flag |= any non-finite w
__global__ void __launch_bounds__(MD_THREADS) k_multidot(int64_t n, const double* __restrict__ V, int64_t ld, int k,
                                                         const double* __restrict__ w, double* __restrict__ out,
                                                         int* flag, MdScratch ms) {
  __shared__ double ws[MD_THREADS / 32];
  __shared__ bool last;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int c0 = 0; c0 < k; c0 += MD_CH) {
    double acc[MD_CH];
#pragma unroll
    for (int c = 0; c < MD_CH; ++c) acc[c] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const double wi = w[i];
      if (c0 == 0 && !isfinite(wi)) bad = true;
#pragma unroll
      for (int c = 0; c < MD_CH; ++c)
        if (c0 + c < k) acc[c] += V[(int64_t)(c0 + c) * ld + i] * wi;
    }
#pragma unroll
    for (int c = 0; c < MD_CH; ++c) {
      if (c0 + c >= k) break;
      const double sblk = block_sum_md(acc[c], ws);
      if (threadIdx.x == 0) ms.partial[(int64_t)blockIdx.x * MD_KMAX + c0 + c] = sblk;
    }
  }
  if (flag != nullptr && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ms.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = 0; c < k; ++c) {
    double v = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
      v += ((volatile double*)ms.partial)[(int64_t)b * MD_KMAX + c];
    v = block_sum_md(v, ws);
    if (threadIdx.x == 0) out[c] = v;
  }
  if (threadIdx.x == 0) *ms.counter = 0u;
}

int launch_multidot(int64_t n, const double* V, int64_t ld, int k, const double* w, double* out, int* flag,
                    cudaStream_t st) {
  if (k < 1 || k > MD_KMAX) return -1001;
  MdScratch ms;
  int e = md_scratch(&ms, st);
  if (e) return e;
  k_multidot<<<MD_BLOCKS, MD_THREADS, 0, st>>>(n, V, ld, k, w, out, flag, ms);
  return (int)cudaGetLastError();
}

// w -= V[0:k]^T y (y on the device; the sum in gemv_t's order, then one
// subtraction)
__global__ void k_gemv_sub(int64_t n, int k, const double* __restrict__ V, int64_t ld, const double* y,
                           double* __restrict__ w) {
  extern __shared__ double ys[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += V[(int64_t)j * ld + i] * ys[j];
    w[i] = w[i] - s;
  }
}

int launch_gemv_sub(int64_t n, int k, const double* V, int64_t ld, const double* y, double* w, cudaStream_t st) {
  if (k < 1 || k > MD_KMAX) return -1001;
  k_gemv_sub<<<ew_grid(n), 256, sizeof(double) * k, st>>>(n, k, V, ld, y, w);
  return (int)cudaGetLastError();
}

}  // namespace pmgb

namespace pmgb {

// FP64 peak probe: 8 independent DFMA chains per thread, full grid.
// flops = 2 * 8 * iters * threads.  Used by bench.py for the FP64 roof
// (MEASURED_PEAKS.json has HBM and bf16 only).
__global__ void __launch_bounds__(256) k_probe_fp64(int64_t iters, double seed, double* out) {
  double a0 = seed + threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
  double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
  const double m = 0.999999999, c = 1e-12;
  for (int64_t i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

int launch_probe_fp64(int64_t iters, int blocks, double* out, cudaStream_t st) {
  k_probe_fp64<<<blocks, 256, 0, st>>>(iters, 1.0, out);
  return (int)cudaGetLastError();
}

}  // namespace pmgb
