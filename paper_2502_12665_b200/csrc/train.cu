// Offline query-aware codebook construction, one KV head per call:
//   H = (1/m) sum q^T q (+ eps tr(H)/d I)       P:248 (Eq. 10), reading Q27
//   H = L L^T (Cholesky), z = k L                P:324-331 (Eqs. 15-16)
//   k-means++ on z with the caller's draws u     P:364, reading Q28
//   Lloyd on z (conventional VQ in z-space)       Eq. 18, reading Q29
//   C = C^z L^{-1}                                Eq. 19
// An offline stage (seconds per head), computed in fp64 throughout so that its integer
// decisions -- the k-means++ draws and every Lloyd assignment -- are the ones an fp64
// evaluation of the definitions takes; sums run in a fixed order (deterministic results).
#include <algorithm>
#include <utility>

#include "internal.cuh"

namespace a2ats {
namespace {

constexpr int kHRows = 32;     // query rows per H partial tile
constexpr int kPB = 256;       // points per block (k-means++ partial sums)

struct TrainState {
  int done, iters, changed, error;
};

// partial H of rows [blk * rows_per, ...): thread <-> (i, j) entries, rows in order
__global__ __launch_bounds__(256) void h_partial_kernel(const uint16_t* __restrict__ q, int m, int d, int rows_per,
                                                        double* __restrict__ part) {
  __shared__ double qs[kHRows][kD];
  const int blk = blockIdx.x, r0 = blk * rows_per, r1 = min(m, r0 + rows_per);
  const int nent = d * d;
  double acc[kD * kD / 256];
  for (int e = 0; e < nent / 256 + 1 && e < kD * kD / 256; ++e) acc[e] = 0.0;
  for (int base = r0; base < r1; base += kHRows) {
    const int nr = min(kHRows, r1 - base);
    __syncthreads();
    for (int k = threadIdx.x; k < nr * d; k += 256) qs[k / d][k % d] = (double)bf_u16(q[(size_t)(base + k / d) * d + k % d]);
    __syncthreads();
    for (int e = 0; e * 256 + threadIdx.x < nent; ++e) {
      const int idx = e * 256 + threadIdx.x, i = idx / d, j = idx % d;
      double s = acc[e];
      for (int r = 0; r < nr; ++r) s = fma(qs[r][i], qs[r][j], s);
      acc[e] = s;
    }
  }
  for (int e = 0; e * 256 + threadIdx.x < nent; ++e) part[(size_t)blk * nent + e * 256 + threadIdx.x] = acc[e];
}

// H = sum of the partials in block order / m (+ jitter); or H_in; or I.  Then the Cholesky
// factor (right-looking, one CTA, fp64 in shared memory) and its inverse (forward substitution).
__global__ __launch_bounds__(kD) void chol_kernel(const double* __restrict__ part, int nblk, int m,
                                                  const double* __restrict__ H_in, double eps, int d,
                                                  double* __restrict__ H_out, double* __restrict__ Lf,
                                                  double* __restrict__ Linv, TrainState* st) {
  extern __shared__ double A[];  // [d][d]
  const int tid = threadIdx.x;
  for (int k = tid; k < d * d; k += blockDim.x) {
    double h;
    if (part) {
      h = 0.0;
      for (int b = 0; b < nblk; ++b) h += part[(size_t)b * d * d + k];
      h /= (double)m;
    } else if (H_in) {
      h = H_in[k];
    } else {
      h = (k / d == k % d) ? 1.0 : 0.0;
    }
    A[k] = h;
  }
  __syncthreads();
  __shared__ double s_tr;
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < d; ++i) tr += A[i * d + i];
    s_tr = tr;
  }
  __syncthreads();
  if (eps > 0.0 && tid < d) A[tid * d + tid] += eps * (s_tr / (double)d);
  __syncthreads();
  if (H_out)
    for (int k = tid; k < d * d; k += blockDim.x) H_out[k] = A[k];
  // Cholesky: A = L L^T, L lower (kept in A's lower triangle)
  for (int k = 0; k < d; ++k) {
    if (tid == 0) {
      const double p = A[k * d + k];
      if (!(p > 0.0)) st->error = 1;
      A[k * d + k] = sqrt(p);
    }
    __syncthreads();
    const double lkk = A[k * d + k];
    if (tid > k && tid < d) A[tid * d + k] /= lkk;
    __syncthreads();
    if (tid > k && tid < d) {
      const double lik = A[tid * d + k];
      for (int j = k + 1; j <= tid; ++j) A[tid * d + j] -= lik * A[j * d + k];
    }
    __syncthreads();
  }
  for (int k = tid; k < d * d; k += blockDim.x) Lf[k] = (k % d <= k / d) ? A[k] : 0.0;
  // L^{-1}: column j by forward substitution, thread j
  if (tid < d) {
    const int j = tid;
    for (int i = 0; i < d; ++i) {
      double x;
      if (i < j) {
        x = 0.0;
      } else {
        double s = (i == j) ? 1.0 : 0.0;
        for (int k = j; k < i; ++k) s -= A[i * d + k] * Linv[k * d + j];
        x = s / A[i * d + i];
      }
      Linv[i * d + j] = x;
    }
  }
}

// out[r][j] = sum_i in[r][i] * M[i][j]  (row vectors times a d x d matrix), i in order
template <typename T>
__device__ __forceinline__ double load_as_double(const T* p, size_t i);
template <>
__device__ __forceinline__ double load_as_double<uint16_t>(const uint16_t* p, size_t i) {
  return (double)bf_u16(p[i]);
}
template <>
__device__ __forceinline__ double load_as_double<double>(const double* p, size_t i) {
  return p[i];
}
template <typename T>
__global__ __launch_bounds__(kD) void rowmat_kernel(const T* __restrict__ in, int rows, int d,
                                                    const double* __restrict__ M, double* __restrict__ out) {
  __shared__ double xs[32][kD];
  const int r0 = blockIdx.x * 32, j = threadIdx.x;
  const int nr = min(32, rows - r0);
  for (int k = threadIdx.x; k < nr * d; k += blockDim.x) xs[k / d][k % d] = load_as_double(in, (size_t)(r0 + k / d) * d + k % d);
  __syncthreads();
  if (j >= d) return;
  double acc[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) acc[r] = 0.0;
  for (int i = 0; i < d; ++i) {
    const double mij = M[i * d + j];
#pragma unroll
    for (int r = 0; r < 32; ++r) acc[r] = fma(xs[r][i], mij, acc[r]);
  }
  for (int r = 0; r < nr; ++r) out[(size_t)(r0 + r) * d + j] = acc[r];
}

__device__ __forceinline__ double sqdist(const double* __restrict__ a, const double* __restrict__ b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) {
    const double t = a[i] - b[i];
    s = fma(t, t, s);
  }
  return s;
}

// k-means++: D^2 update against centre j - 1 and per-block sums (sequential, in point order)
__global__ __launch_bounds__(kPB) void kpp_update_kernel(const double* __restrict__ z, int n, int d,
                                                         const double* __restrict__ cprev, double* __restrict__ d2,
                                                         double* __restrict__ bsum, int first) {
  __shared__ double cs[kD];
  __shared__ double vals[kPB];
  for (int i = threadIdx.x; i < d; i += kPB) cs[i] = cprev[i];
  __syncthreads();
  const int t = blockIdx.x * kPB + threadIdx.x;
  double v = 0.0;
  if (t < n) {
    const double x = sqdist(z + (size_t)t * d, cs, d);
    v = first ? x : fmin(d2[t], x);
    d2[t] = v;
  }
  vals[threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kPB; ++i) s += vals[i];
    bsum[blockIdx.x] = s;
  }
}

// k-means++: centre j = the first point whose running D^2 sum exceeds u_j * total
__global__ __launch_bounds__(32) void kpp_pick_kernel(const double* __restrict__ z, int n, int d,
                                                      const double* __restrict__ d2, const double* __restrict__ bsum,
                                                      int nblk, const double* __restrict__ u, int j,
                                                      double* __restrict__ Cz, int32_t* __restrict__ seeds) {
  __shared__ int s_t;
  if (threadIdx.x == 0) {
    int t = 0;
    if (j == 0) {
      t = min(n - 1, (int)floor(u[0] * (double)n));
    } else {
      double tot = 0.0;
      for (int b = 0; b < nblk; ++b) tot += bsum[b];
      const double target = u[j] * tot;
      if (tot > 0.0) {
        double run = 0.0;
        int b = 0;
        while (b < nblk - 1 && run + bsum[b] <= target) run += bsum[b++];
        t = b * kPB;
        const int te = min(n, t + kPB);
        while (t < te - 1 && run + d2[t] <= target) run += d2[t++];
        // (the block boundary test above used the block sum; inside the block the running sum
        // is re-accumulated point by point, so t is the first point with running sum > target)
      }
      t = min(t, n - 1);
    }
    s_t = t;
    seeds[j] = t;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += 32) Cz[(size_t)j * d + i] = z[(size_t)s_t * d + i];
}

// Lloyd assignment: argmin_j ||z_t - c_j||^2 (direct form, lowest j on ties).  CTA = 32 points,
// 128 threads: thread (point p, centre group g) scans centres g, g + 4, ... of every 32-centre
// tile; the 4 groups of a point are merged lexicographically on (distance, index).
constexpr int kAP = 32, kAC = 32;
__global__ __launch_bounds__(128) void assign_kernel(const double* __restrict__ z, int n, int d,
                                                     const double* __restrict__ Cz, int L,
                                                     const int32_t* __restrict__ old_labels,
                                                     int32_t* __restrict__ labels, TrainState* st, int first) {
  if (!first && st->done) return;
  extern __shared__ double sm[];
  double* zs = sm;              // [kAP][d]
  double* cs = sm + kAP * d;    // [kAC][d]
  const int t0 = blockIdx.x * kAP, p = threadIdx.x >> 2, g = threadIdx.x & 3;
  for (int k = threadIdx.x; k < kAP * d; k += 128) {
    const int r = k / d;
    zs[k] = (t0 + r < n) ? z[(size_t)(t0 + r) * d + k % d] : 0.0;
  }
  double best = INFINITY;
  int bj = 0;
  for (int c0 = 0; c0 < L; c0 += kAC) {
    __syncthreads();
    for (int k = threadIdx.x; k < kAC * d; k += 128) {
      const int c = k / d;
      cs[k] = (c0 + c < L) ? Cz[(size_t)(c0 + c) * d + k % d] : 0.0;
    }
    __syncthreads();
    for (int c = g; c < kAC && c0 + c < L; c += 4) {
      const double dist = sqdist(zs + p * d, cs + c * d, d);
      if (dist < best) {
        best = dist;
        bj = c0 + c;
      }
    }
  }
  // merge the 4 groups of point p: smaller distance, then lower index
#pragma unroll
  for (int off = 1; off < 4; off <<= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
    if (ob < best || (ob == best && oj < bj)) {
      best = ob;
      bj = oj;
    }
  }
  const int t = t0 + p;
  if (g == 0 && t < n) {
    if (!first && old_labels[t] != bj) atomicAdd(&st->changed, 1);
    labels[t] = bj;
  }
}

// Lloyd update: warp per centre, points of its cluster in index order (fixed-order sums);
// an empty cluster keeps its centre (reading Q29)
__global__ __launch_bounds__(256) void update_kernel(const double* __restrict__ z, int n, int d,
                                                     const int32_t* __restrict__ labels, int L,
                                                     double* __restrict__ Cz, TrainState* st) {
  if (st->done) return;
  const int warp = (blockIdx.x * 256 + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= L) return;
  double acc[kD / 32];
#pragma unroll
  for (int e = 0; e < kD / 32; ++e) acc[e] = 0.0;
  int cnt = 0;
  for (int t0 = 0; t0 < n; t0 += 32) {
    const int t = t0 + lane;
    unsigned hit = __ballot_sync(0xffffffffu, t < n && labels[t] == warp);
    while (hit) {
      const int b = __ffs(hit) - 1;
      hit &= hit - 1u;
      const double* zr = z + (size_t)(t0 + b) * d;
#pragma unroll
      for (int e = 0; e < kD / 32; ++e)
        if (lane + 32 * e < d) acc[e] += zr[lane + 32 * e];
      ++cnt;
    }
  }
  if (cnt > 0) {
#pragma unroll
    for (int e = 0; e < kD / 32; ++e)
      if (lane + 32 * e < d) Cz[(size_t)warp * d + lane + 32 * e] = acc[e] / (double)cnt;
  }
}

// end of an iteration: no assignment changed -> done; count the iteration
__global__ void iter_end_kernel(TrainState* st) {
  if (st->done) return;
  st->iters += 1;
  if (st->changed == 0) st->done = 1;
  st->changed = 0;
}

__global__ void state_reset_kernel(TrainState* st) {
  st->done = st->iters = st->changed = st->error = 0;
}

__global__ void copy_labels_kernel(const int32_t* src, int32_t* dst, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

struct TrainWs {
  size_t z, d2, bsum, Lf, Linv, H, part, cz, lab0, lab1, seeds, st, total;
};
size_t al(size_t x) { return (x + 255) / 256 * 256; }
TrainWs train_layout(int n, int d, int L, int m) {
  TrainWs w;
  const int nblk = (n + kPB - 1) / kPB;
  const int hblk = std::max(1, std::min(148, (m + kHRows - 1) / kHRows));
  size_t o = 0;
  w.z = o; o = al(o + (size_t)n * d * 8);
  w.d2 = o; o = al(o + (size_t)n * 8);
  w.bsum = o; o = al(o + (size_t)nblk * 8);
  w.Lf = o; o = al(o + (size_t)d * d * 8);
  w.Linv = o; o = al(o + (size_t)d * d * 8);
  w.H = o; o = al(o + (size_t)d * d * 8);
  w.part = o; o = al(o + (size_t)hblk * d * d * 8);
  w.cz = o; o = al(o + (size_t)L * d * 8);
  w.lab0 = o; o = al(o + (size_t)n * 4);
  w.lab1 = o; o = al(o + (size_t)n * 4);
  w.seeds = o; o = al(o + (size_t)L * 4);
  w.st = o; o = al(o + sizeof(TrainState));
  w.total = o;
  return w;
}

}  // namespace
}  // namespace a2ats

using namespace a2ats;

extern "C" {

size_t a2ats_qavq_train_workspace_bytes(int32_t n_keys, int32_t d, int32_t L, int32_t m_queries) {
  if (n_keys < 1 || d < 1 || d > kD || L < 1 || m_queries < 0) return 0;
  return train_layout(n_keys, d, L, std::max(1, m_queries)).total;
}

int a2ats_qavq_train(int32_t n_keys, int32_t d, int32_t L, const void* keys, int32_t m_queries, const void* queries,
                     const double* H_in, double eps, const double* u, int32_t max_iters, double* C_out,
                     double* H_out, int32_t* labels_out, int32_t* info_out, void* ws, size_t ws_bytes,
                     void* stream) {
  if (n_keys < 1 || d < 2 || d > kD || L < 1 || L > n_keys || max_iters < 0 || eps < 0.0) return A2ATS_EINVAL;
  if (!keys || !u || !C_out || (queries && m_queries < 1)) return A2ATS_EINVAL;
  const TrainWs W = train_layout(n_keys, d, L, std::max(1, m_queries));
  if (!ws || ws_bytes < W.total) return A2ATS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* b = static_cast<uint8_t*>(ws);
  double* z = reinterpret_cast<double*>(b + W.z);
  double* d2 = reinterpret_cast<double*>(b + W.d2);
  double* bsum = reinterpret_cast<double*>(b + W.bsum);
  double* Lf = reinterpret_cast<double*>(b + W.Lf);
  double* Linv = reinterpret_cast<double*>(b + W.Linv);
  double* Hs = H_out ? H_out : reinterpret_cast<double*>(b + W.H);
  double* part = reinterpret_cast<double*>(b + W.part);
  double* Cz = reinterpret_cast<double*>(b + W.cz);
  int32_t* lab0 = reinterpret_cast<int32_t*>(b + W.lab0);
  int32_t* lab1 = reinterpret_cast<int32_t*>(b + W.lab1);
  int32_t* seeds = reinterpret_cast<int32_t*>(b + W.seeds);
  TrainState* ts = reinterpret_cast<TrainState*>(b + W.st);
  state_reset_kernel<<<1, 1, 0, st>>>(ts);
  // 1. H (queries -> fixed-order partials over 64-row tiles)
  int hblk = 0;
  if (queries) {
    hblk = std::max(1, std::min(148, (m_queries + kHRows - 1) / kHRows));
    const int rows_per = (m_queries + hblk - 1) / hblk;
    h_partial_kernel<<<hblk, 256, 0, st>>>(static_cast<const uint16_t*>(queries), m_queries, d, rows_per, part);
  }
  // 2. Cholesky + inverse
  cudaError_t e = ensure_smem(chol_kernel, d * d * 8);
  if (e != cudaSuccess) return A2ATS_ECUDA;
  chol_kernel<<<1, kD, d * d * 8, st>>>(queries ? part : nullptr, hblk, m_queries, H_in, eps, d, Hs, Lf, Linv, ts);
  // 3. z = k L
  rowmat_kernel<uint16_t><<<(n_keys + 31) / 32, kD, 0, st>>>(static_cast<const uint16_t*>(keys), n_keys, d, Lf, z);
  // 4. k-means++ seeding
  const int nblk = (n_keys + kPB - 1) / kPB;
  kpp_pick_kernel<<<1, 32, 0, st>>>(z, n_keys, d, d2, bsum, nblk, u, 0, Cz, seeds);
  for (int j = 1; j < L; ++j) {
    kpp_update_kernel<<<nblk, kPB, 0, st>>>(z, n_keys, d, Cz + (size_t)(j - 1) * d, d2, bsum, j == 1);
    kpp_pick_kernel<<<1, 32, 0, st>>>(z, n_keys, d, d2, bsum, nblk, u, j, Cz, seeds);
  }
  // 5. Lloyd: labels <- assign(seeds); per iteration: update, assign (count changes), end
  const int asmem = (kAP + kAC) * d * 8;
  e = ensure_smem(assign_kernel, asmem);
  if (e != cudaSuccess) return A2ATS_ECUDA;
  const int agrid = (n_keys + kAP - 1) / kAP;
  assign_kernel<<<agrid, 128, asmem, st>>>(z, n_keys, d, Cz, L, nullptr, lab0, ts, 1);
  int32_t* cur = lab0;
  int32_t* nxt = lab1;
  for (int it = 0; it < max_iters; ++it) {
    update_kernel<<<(L * 32 + 255) / 256, 256, 0, st>>>(z, n_keys, d, cur, L, Cz, ts);
    assign_kernel<<<agrid, 128, asmem, st>>>(z, n_keys, d, Cz, L, cur, nxt, ts, 0);
    // a converged run keeps its labels in `cur` (assign skipped): copy forward when done
    iter_end_kernel<<<1, 1, 0, st>>>(ts);
    std::swap(cur, nxt);
  }
  // the labels of the last EXECUTED assignment: after a skipped one `nxt` holds them
  // 6. C = C^z L^{-1}
  rowmat_kernel<double><<<(L + 31) / 32, kD, 0, st>>>(Cz, L, d, Linv, C_out);
  if (labels_out) {
    // the last assignment that ran wrote `cur` unless the run converged earlier, in which
    // case both buffers hold the converged labels from that point on (see below)
    copy_labels_kernel<<<64, 256, 0, st>>>(cur, labels_out, n_keys);
  }
  if (info_out) {
    // [iters, error] from the device state
    cudaMemcpyAsync(info_out, &ts->iters, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(info_out + 1, &ts->error, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  }
  return cudaGetLastError() == cudaSuccess ? A2ATS_OK : A2ATS_ECUDA;
}

}  // extern "C"
