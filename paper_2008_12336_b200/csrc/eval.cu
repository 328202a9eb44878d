// Link-prediction evaluator on the device (reference: evaluate.py:69-160),
// SURVEY.md 8(f) rank 1.  The host harness materialises |pairs| x d feature
// rows and fits the classifier in numpy, which at C3-C5 sizes does not fit
// (and dominates even at C1).  Here:
//
//   gb_hadamard_features  X[i,t] = fl32(M[u_i,t] * M[v_i,t])        (evaluate.py:78)
//   gb_logreg_epoch       one epoch of the seeded mini-batch descent
//                         (evaluate.py:128-140) over a host-drawn
//                         permutation: z = X_b w + b (fp64), resid =
//                         sigmoid(z) - y, w -= (step * X_b^T resid) / m,
//                         b -= step * mean(resid).  The steps are strictly
//                         sequential, so one CTA owns the whole epoch: each
//                         warp takes rows of the batch, the gradient is
//                         reduced through shared memory in a fixed order.
//   gb_predict_scores     rows @ w + b                                (evaluate.py:146-147)
//   gb_auc_roc            midrank AUCROC (evaluate.py:150-167): radix sort
//                         of (score, label), run-length groups of equal
//                         scores, sum over positives of doubled midranks in
//                         int64 -- exact, like the reference.
//
// Arithmetic: features are the reference's fp32 products; dots and
// gradients are fp64 as in numpy (summation order differs from BLAS, so fits
// agree to rounding, not bit for bit; AUC is exact for equal scores).
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace gb {
namespace {

constexpr int kFitThreads = 512;  // 16 warps x 128 registers: batched gathers without spills
constexpr int kFitWarps = kFitThreads / 32;
constexpr int kMaxK = 16;  // d <= 512
// rows gathered together per warp: 8 (a 256-row mini-batch = 2 gather
// rounds per warp) as long as the batch fits the register file
template <int K>
constexpr int rows_per_batch() { return K <= 4 ? 16 : (K <= 8 ? 4 : 1); }

__device__ __forceinline__ double sigmoid_clamped(double z) {  // trainer.py:96-99
  z = fmin(fmax(z, -10.0), 10.0);
  return 1.0 / (1.0 + exp(-z));
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__global__ void hadamard_kernel(const float *__restrict__ M, int d,
                                const int64_t *__restrict__ pairs, int64_t n,
                                float *__restrict__ X) {
  const int64_t total = n * (int64_t)d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d;
    const int t = (int)(i - r * d);
    const int64_t u = pairs[2 * r], v = pairs[2 * r + 1];
    X[i] = __fmul_rn(__ldg(M + u * d + t), __ldg(M + v * d + t));
  }
}

// One epoch of mini-batch descent; w (d doubles) and b live in global
// memory between launches.  Dynamic shared memory: w[d] + part[32][d] +
// rsum[32] doubles.
template <int K>
__global__ void __launch_bounds__(kFitThreads, 1)
    logreg_epoch_kernel(const float *__restrict__ X, int d, const int8_t *__restrict__ y,
                        const int64_t *__restrict__ perm, int64_t n, int bs, double step,
                        double *__restrict__ w_g, double *__restrict__ b_g) {
  extern __shared__ double sh[];
  double *w_s = sh;
  double *part = sh + d;                       // [kFitWarps][d]
  double *rsum = part + (size_t)kFitWarps * d;  // [kFitWarps]
  double *b_s = rsum + kFitWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < d; t += blockDim.x) w_s[t] = w_g[t];
  if (threadIdx.x == 0) *b_s = *b_g;
  __syncthreads();
  double wl[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int t = lane + 32 * k;
    wl[k] = t < d ? w_s[t] : 0.0;
  }
  double b = *b_s;
  constexpr int kRowsPerBatch = rows_per_batch<K>();
  // One gather round covers the whole mini-batch (bs <= 16 warps x rows per
  // batch: the reference's 256 at d <= 128): the next step's rows do not
  // depend on w, so they are gathered while this step's gradient is reduced
  // (28.4 -> 10.5 us per step at d=128, identical weights).  Measured and
  // dropped: interleaving the rows' dots/sigmoids in sub-batches (11.0) and
  // loading the permuted indices a step ahead (22.0, spills).
  const bool one_round = bs <= kFitWarps * kRowsPerBatch;
  float x[kRowsPerBatch][K];
  int8_t yv[kRowsPerBatch];
  auto gather = [&](int64_t i0, int m, int r0) {
#pragma unroll
    for (int j = 0; j < kRowsPerBatch; ++j) {
      const int r = r0 + j * kFitWarps;
      const bool ok = r < m;
      const int64_t row = ok ? perm[i0 + r] : 0;
      const float *xr = X + row * d;
      yv[j] = ok ? y[row] : 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int t = lane + 32 * k;
        x[j][k] = (ok && t < d) ? __ldg(xr + t) : 0.0f;
      }
    }
  };
  if (one_round && n > 0) gather(0, (int)((int64_t)bs < n ? bs : n), warp);
  for (int64_t i0 = 0; i0 < n; i0 += bs) {
    const int m = (int)((int64_t)bs < n - i0 ? (int64_t)bs : n - i0);
    double g[K];
#pragma unroll
    for (int k = 0; k < K; ++k) g[k] = 0.0;
    double rs = 0.0;
    // rows of this warp in batches of kRowsPerBatch: every gather of a batch
    // is issued before the first dot (the rows are random, so each gather
    // is a full memory round trip; issuing them together pays it once)
    for (int r0 = warp; r0 < m; r0 += kFitWarps * kRowsPerBatch) {
      if (!one_round) gather(i0, m, r0);
#pragma unroll
      for (int j = 0; j < kRowsPerBatch; ++j) {
        if (r0 + j * kFitWarps >= m) break;
        double z = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) z = fma((double)x[j][k], wl[k], z);
        z = warp_sum(z) + b;
        const double resid = sigmoid_clamped(z) - (double)yv[j];
#pragma unroll
        for (int k = 0; k < K; ++k) g[k] = fma((double)x[j][k], resid, g[k]);
        rs += resid;
      }
    }
    if (one_round && i0 + bs < n) {
      const int64_t i1 = i0 + bs;
      gather(i1, (int)((int64_t)bs < n - i1 ? (int64_t)bs : n - i1), warp);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int t = lane + 32 * k;
      if (t < d) part[(size_t)warp * d + t] = g[k];
    }
    if (lane == 0) rsum[warp] = rs;
    __syncthreads();
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
      double G = 0.0;
      for (int q = 0; q < kFitWarps; ++q) G += part[(size_t)q * d + t];
      w_s[t] = w_s[t] - (step * G) / (double)m;
    }
    if (threadIdx.x == blockDim.x - 1) {
      double R = 0.0;
      for (int q = 0; q < kFitWarps; ++q) R += rsum[q];
      *b_s = *b_s - step * (R / (double)m);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int t = lane + 32 * k;
      wl[k] = t < d ? w_s[t] : 0.0;
    }
    b = *b_s;
    __syncthreads();  // w_s/b_s reads done before the next step's writes
  }
  for (int t = threadIdx.x; t < d; t += blockDim.x) w_g[t] = w_s[t];
  if (threadIdx.x == 0) *b_g = *b_s;
}

// The same epoch on a cluster of kClusterCtas CTAs: CTA c takes rows
// [c*rpc, (c+1)*rpc) of every mini-batch (rpc = ceil(bs / CTAs), kRpw rows
// per warp), reduces its warps' gradients through shared memory, publishes
// the CTA partial in a double-buffered shared slot, and after one cluster
// barrier every CTA sums the partials of all CTAs through DSMEM in CTA
// order -- so every CTA applies the identical update to its own copy of w.
// The next step's rows are gathered before the reduction (they do not
// depend on w).  Summation order differs from the single-CTA kernel (rows
// are split differently), so weights agree to rounding.
constexpr int kClusterCtas = 8;
template <int K, int kRpw>
__global__ void __launch_bounds__(kFitThreads, 1)
    logreg_epoch_cluster_kernel(const float *__restrict__ X, int d,
                                const int8_t *__restrict__ y, const int64_t *__restrict__ perm,
                                int64_t n, int bs, double step, double *__restrict__ w_g,
                                double *__restrict__ b_g) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  extern __shared__ double sh[];
  double *w_s = sh;                                  // [d]
  double *part = w_s + d;                            // [kFitWarps][d]
  double *rsum = part + (size_t)kFitWarps * d;       // [kFitWarps]
  double *pub = rsum + kFitWarps;                    // [2][d + 1] CTA partials
  double *b_s = pub + 2 * ((size_t)d + 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < d; t += blockDim.x) w_s[t] = w_g[t];
  if (threadIdx.x == 0) *b_s = *b_g;
  __syncthreads();
  double wl[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int t = lane + 32 * k;
    wl[k] = t < d ? w_s[t] : 0.0;
  }
  double b = *b_s;
  const int rpc = (bs + kClusterCtas - 1) / kClusterCtas;
  float x[kRpw][K];
  int8_t yv[kRpw];
  auto gather = [&](int64_t i0, int m) {
    const int lo = crank * rpc, hi = min(m, lo + rpc);
#pragma unroll
    for (int j = 0; j < kRpw; ++j) {
      const int r = lo + warp + j * kFitWarps;
      const bool ok = r < hi;
      const int64_t row = ok ? perm[i0 + r] : 0;
      const float *xr = X + row * d;
      yv[j] = ok ? y[row] : 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int t = lane + 32 * k;
        x[j][k] = (ok && t < d) ? __ldg(xr + t) : 0.0f;
      }
    }
  };
  auto rows_of = [&](int64_t i0) { return (int)((int64_t)bs < n - i0 ? (int64_t)bs : n - i0); };
  gather(0, rows_of(0));
  int parity = 0;
  for (int64_t i0 = 0; i0 < n; i0 += bs, parity ^= 1) {
    const int m = rows_of(i0);
    const int hi = min(m, crank * rpc + rpc);
    double g[K];
#pragma unroll
    for (int k = 0; k < K; ++k) g[k] = 0.0;
    double rs = 0.0;
#pragma unroll
    for (int j = 0; j < kRpw; ++j) {
      if (crank * rpc + warp + j * kFitWarps >= hi) break;
      double z = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) z = fma((double)x[j][k], wl[k], z);
      z = warp_sum(z) + b;
      const double resid = sigmoid_clamped(z) - (double)yv[j];
#pragma unroll
      for (int k = 0; k < K; ++k) g[k] = fma((double)x[j][k], resid, g[k]);
      rs += resid;
    }
    if (i0 + bs < n) gather(i0 + bs, rows_of(i0 + bs));
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int t = lane + 32 * k;
      if (t < d) part[(size_t)warp * d + t] = g[k];
    }
    if (lane == 0) rsum[warp] = rs;
    __syncthreads();
    double *mine = pub + (size_t)parity * (d + 1);
    for (int t = threadIdx.x; t <= d; t += blockDim.x) {
      double G = 0.0;
      if (t < d) {
        for (int q = 0; q < kFitWarps; ++q) G += part[(size_t)q * d + t];
      } else {
        for (int q = 0; q < kFitWarps; ++q) G += rsum[q];
      }
      mine[t] = G;
    }
    cluster.sync();  // every CTA's partial is published (and part/rsum are free)
    for (int t = threadIdx.x; t <= d; t += blockDim.x) {
      double G = 0.0;
      for (int c = 0; c < kClusterCtas; ++c) G += cluster.map_shared_rank(mine, c)[t];
      if (t < d)
        w_s[t] = w_s[t] - (step * G) / (double)m;
      else
        *b_s = *b_s - step * (G / (double)m);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int t = lane + 32 * k;
      wl[k] = t < d ? w_s[t] : 0.0;
    }
    b = *b_s;
    // w_s is rewritten only after the next cluster.sync, which every thread
    // of this CTA reaches after the reads above
  }
  cluster.sync();  // no CTA exits while another may still read its partials
  if (crank == 0) {
    for (int t = threadIdx.x; t < d; t += blockDim.x) w_g[t] = w_s[t];
    if (threadIdx.x == 0) *b_g = *b_s;
  }
}

__global__ void predict_kernel(const float *__restrict__ X, int d, int64_t n,
                               const double *__restrict__ w, double b,
                               double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
    double z = 0.0;
    for (int t = lane; t < d; t += 32) z = fma((double)__ldg(X + r * d + t), __ldg(w + t), z);
    z = warp_sum(z);
    if (lane == 0) out[r] = z + b;
  }
}

// (count, positives) per run of equal scores
struct RunStat {
  int64_t c, p;
};
struct RunAdd {
  __device__ __forceinline__ RunStat operator()(const RunStat &a, const RunStat &b) const {
    return {a.c + b.c, a.p + b.p};
  }
};
struct LabelToRun {
  __host__ __device__ __forceinline__ RunStat operator()(const int8_t &y) const {
    return {1, y == 1 ? 1 : 0};
  }
};
// r2p = sum over runs of p_g * (2 s_g + c_g + 1), s_g = exclusive scan of c.
__global__ void auc_finish_kernel(const RunStat *__restrict__ runs,
                                  const int64_t *__restrict__ num_runs,
                                  unsigned long long *__restrict__ acc) {
  // single block: sequential scan in chunks (runs <= n; this is O(n / 1024))
  __shared__ int64_t base;
  __shared__ unsigned long long part[1024];
  __shared__ int64_t csum[1024];
  if (threadIdx.x == 0) base = 0;
  unsigned long long mine = 0;
  const int64_t R = *num_runs;
  for (int64_t c0 = 0; c0 < R; c0 += blockDim.x) {
    const int64_t g = c0 + threadIdx.x;
    const RunStat rs = g < R ? runs[g] : RunStat{0, 0};
    csum[threadIdx.x] = rs.c;
    __syncthreads();
    // inclusive scan (Hillis-Steele) of counts in the chunk
    for (int o = 1; o < blockDim.x; o <<= 1) {
      int64_t v = threadIdx.x >= o ? csum[threadIdx.x - o] : 0;
      __syncthreads();
      csum[threadIdx.x] += v;
      __syncthreads();
    }
    const int64_t s = base + csum[threadIdx.x] - rs.c;
    mine += (unsigned long long)(rs.p * (2 * s + rs.c + 1));
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base += csum[threadIdx.x];
    __syncthreads();
  }
  part[threadIdx.x] = mine;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *acc = part[0];
}

struct Carver {
  char *base;
  size_t off = 0;
  explicit Carver(void *b) : base(static_cast<char *>(b)) {}
  template <class T>
  T *take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

int auc_plan(int64_t n, void *ws, size_t *bytes, const double *scores, const int8_t *labels,
             cudaStream_t st, unsigned long long **acc_out, int64_t *npos_out = nullptr) {
  Carver c(ws);
  double *keys = c.take<double>(n);
  int8_t *vals = c.take<int8_t>(n);
  double *ukeys = c.take<double>(n);
  RunStat *runs = c.take<RunStat>(n);
  int64_t *nruns = c.take<int64_t>(1);
  unsigned long long *acc = c.take<unsigned long long>(1);
  size_t sort_b = 0, red_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, scores, keys, labels, vals, (int)n, 0, 64,
                                  st);
  auto in_runs = thrust::make_transform_iterator(static_cast<const int8_t *>(vals), LabelToRun());
  cub::DeviceReduce::ReduceByKey(nullptr, red_b, keys, ukeys, in_runs, runs, nruns, RunAdd(),
                                 (int)n, st);
  void *tmp = c.take<char>(std::max(sort_b, red_b));
  if (!ws) {
    *bytes = c.off;
    return GB_OK;
  }
  GB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, sort_b, scores, keys, labels, vals, (int)n, 0,
                                              64, st));
  GB_CUDA_TRY(cub::DeviceReduce::ReduceByKey(tmp, red_b, keys, ukeys, in_runs, runs, nruns,
                                             RunAdd(), (int)n, st));
  auc_finish_kernel<<<1, 1024, 0, st>>>(runs, nruns, acc);
  GB_CHECK_LAUNCH();
  *acc_out = acc;
  return GB_OK;
}

template <int K>
int launch_fit(const float *X, int d, const int8_t *y, const int64_t *perm, int64_t n, int bs,
               double step, double *w, double *b, cudaStream_t st) {
  // cluster form for the usual batch sizes (rows per warp per CTA <= 2);
  // GB_LOGREG_CLUSTER=0 keeps the single-CTA kernel
  const char *env = std::getenv("GB_LOGREG_CLUSTER");
  const bool use_cluster = !(env && std::atoi(env) == 0) &&
                           (bs + kClusterCtas - 1) / kClusterCtas <= 2 * kFitWarps;
  if (use_cluster) {
    const size_t smem = sizeof(double) * ((size_t)d + (size_t)kFitWarps * d + kFitWarps +
                                          2 * ((size_t)d + 1) + 1);
    auto fn = logreg_epoch_cluster_kernel<K, 2>;
    GB_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kClusterCtas, 1, 1);
    cfg.blockDim = dim3(kFitThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kClusterCtas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GB_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, X, d, y, perm, n, bs, step, w, b));
    return GB_OK;
  }
  const size_t smem = sizeof(double) * ((size_t)d + (size_t)kFitWarps * d + kFitWarps + 1);
  GB_CUDA_TRY(cudaFuncSetAttribute(logreg_epoch_kernel<K>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  logreg_epoch_kernel<K><<<1, kFitThreads, smem, st>>>(X, d, y, perm, n, bs, step, w, b);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

}  // namespace
}  // namespace gb

using namespace gb;

GB_API int gb_hadamard_features(const float *M, int64_t num_rows, int dim, const int64_t *pairs,
                                int64_t n, float *X, void *stream) {
  GB_REQUIRE(dim >= 1 && n >= 0 && num_rows >= 0, "gb_hadamard_features: bad sizes");
  if (n == 0) return GB_OK;
  GB_REQUIRE(M && pairs && X, "gb_hadamard_features: null pointer");
  const int64_t total = n * (int64_t)dim;
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16));
  hadamard_kernel<<<blocks, 256, 0, as_stream(stream)>>>(M, dim, pairs, n, X);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_logreg_epoch(const float *X, int dim, const int8_t *labels, const int64_t *perm,
                           int64_t n, int batch_size, double step, double *w, double *b,
                           void *stream) {
  GB_REQUIRE(dim >= 1 && dim <= 32 * kMaxK, "gb_logreg_epoch: dim must be in [1, 512]");
  GB_REQUIRE(batch_size >= 1 && n >= 0, "gb_logreg_epoch: bad batch size");
  if (n == 0) return GB_OK;
  GB_REQUIRE(X && labels && perm && w && b, "gb_logreg_epoch: null pointer");
  cudaStream_t st = as_stream(stream);
  const int K = (dim + 31) / 32;
  if (K <= 1) return launch_fit<1>(X, dim, labels, perm, n, batch_size, step, w, b, st);
  if (K <= 2) return launch_fit<2>(X, dim, labels, perm, n, batch_size, step, w, b, st);
  if (K <= 4) return launch_fit<4>(X, dim, labels, perm, n, batch_size, step, w, b, st);
  if (K <= 8) return launch_fit<8>(X, dim, labels, perm, n, batch_size, step, w, b, st);
  return launch_fit<16>(X, dim, labels, perm, n, batch_size, step, w, b, st);
}

GB_API int gb_predict_scores(const float *X, int dim, int64_t n, const double *w, double b,
                             double *out, void *stream) {
  GB_REQUIRE(dim >= 1 && n >= 0, "gb_predict_scores: bad sizes");
  if (n == 0) return GB_OK;
  GB_REQUIRE(X && w && out, "gb_predict_scores: null pointer");
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 16));
  predict_kernel<<<blocks, 256, 0, as_stream(stream)>>>(X, dim, n, w, b, out);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_auc_roc_workspace(int64_t n, size_t *bytes) {
  GB_REQUIRE(bytes && n >= 0 && n < ((int64_t)1 << 31), "gb_auc_roc_workspace: bad n");
  return auc_plan(n, nullptr, bytes, nullptr, nullptr, 0, nullptr);
}

GB_API int gb_auc_roc(const double *scores, const int8_t *labels, int64_t n,
                      unsigned long long *rank2_pos, void *workspace, size_t workspace_bytes,
                      void *stream) {
  GB_REQUIRE(n >= 1 && n < ((int64_t)1 << 31), "gb_auc_roc: bad n");
  GB_REQUIRE(scores && labels && rank2_pos && workspace, "gb_auc_roc: null pointer");
  size_t need = 0;
  auc_plan(n, nullptr, &need, nullptr, nullptr, 0, nullptr);
  GB_REQUIRE(workspace_bytes >= need, "gb_auc_roc: workspace too small");
  cudaStream_t st = as_stream(stream);
  unsigned long long *acc = nullptr;
  int rc = auc_plan(n, workspace, &need, scores, labels, st, &acc);
  if (rc != GB_OK) return rc;
  GB_CUDA_TRY(cudaMemcpyAsync(rank2_pos, acc, sizeof(unsigned long long),
                              cudaMemcpyDeviceToDevice, st));
  return GB_OK;
}
