// a0: query-aware VQ encoding of keys (Eq. 14; Eq. 20).
//
//   f'(k; C) = argmin_j (k - c_j) H (k - c_j)^T = argmin_j ( n_j - 2 (k H) . c_j )
// with n_j = c_j H c_j^T (a2ats_qavq_prepare) because H is symmetric.  The
// kernel therefore (1) maps each key to u = k H (d x d, cheap), then (2) runs
// the same codeword-tile GEMM as the LUT against the bf16 codebook with an
// argmin epilogue.  Ties resolve to the lowest codeword index (reading Q12):
// lexicographic (dist, index) minimum, which is order independent, so the
// split over codeword ranges and the cross-CTA reduction (64-bit atomicMax on
// the complemented (ordered dist, index) word) are deterministic.
#include "internal.cuh"

namespace a2ats {

namespace {
constexpr int kTC = 128, kTV = 64, kCS = kTC + 4, kVS = kTV + 4;
constexpr int kEncSmem = (kD * kCS + kD * kVS) * 4;

// n_j = c_j H c_j^T, one warp per codeword.
__global__ __launch_bounds__(256) void prepare_kernel(const uint16_t* __restrict__ codebook, const float* __restrict__ H,
                                                      float* __restrict__ nrm, int L) {
  extern __shared__ __align__(16) float Hs[];  // [128][128] or unused
  __shared__ float crow[8][kD];
  const int h = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (H) {
    const float4* src = reinterpret_cast<const float4*>(H + (size_t)h * kD * kD);
    for (int i = tid; i < kD * kD / 4; i += 256) reinterpret_cast<float4*>(Hs)[i] = src[i];
  }
  __syncthreads();
  for (int c = blockIdx.x * 64 + warp; c < min(L, blockIdx.x * 64 + 64); c += 8) {
    const uint16_t* cp = codebook + ((size_t)h * L + c) * kD;
#pragma unroll
    for (int i = 0; i < 4; ++i) crow[warp][lane + 32 * i] = bf_u16(cp[lane + 32 * i]);
    __syncwarp();
    float part = 0.f;
    if (H) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = lane + 32 * k;
        float De = 0.f;
        for (int d = 0; d < kD; ++d) De = fmaf(crow[warp][d], Hs[d * kD + e], De);
        part = fmaf(De, crow[warp][e], part);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) part = fmaf(crow[warp][lane + 32 * k], crow[warp][lane + 32 * k], part);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if (lane == 0) nrm[(size_t)h * L + c] = part;
    __syncwarp();
  }
}

// u[h][v] = k[b][h][t] H[h]  (v = b*T + (t - t_begin)), or u = k when H == nullptr.
__global__ __launch_bounds__(256) void keyh_kernel(EncArgs a) {
  extern __shared__ __align__(16) float Hs[];  // [128][128]
  __shared__ float ks[32][kD];
  const int h = blockIdx.y, tid = threadIdx.x;
  const int v0 = blockIdx.x * 32;
  if (a.H) {
    const float4* src = reinterpret_cast<const float4*>(a.H + (size_t)h * kD * kD);
    for (int i = tid; i < kD * kD / 4; i += 256) reinterpret_cast<float4*>(Hs)[i] = src[i];
  }
  for (int i = tid; i < 32 * kD; i += 256) {
    const int vv = i >> 7, d = i & (kD - 1);
    const int v = v0 + vv;
    float x = 0.f;
    if (v < a.nvec) {
      const int b = v / a.T, t = a.t_begin + (v - (v / a.T) * a.T);
      x = bf_u16(a.keys[(((size_t)b * a.Hkv + h) * a.n_max + t) * kD + d]);
    }
    ks[vv][d] = x;
  }
  __syncthreads();
  const int e = tid & (kD - 1), vh = tid >> 7;  // 2 halves of 16 vectors
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  if (a.H) {
#pragma unroll 4
    for (int d = 0; d < kD; ++d) {
      const float hd = Hs[d * kD + e];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(ks[vh * 16 + i][d], hd, acc[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = ks[vh * 16 + i][e];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int v = v0 + vh * 16 + i;
    if (v < a.nvec) a.u[((size_t)h * a.nvec + v) * kD + e] = acc[i];
  }
}

__device__ __forceinline__ unsigned long long pack_dist(float dist, int code) {
  return ((unsigned long long)ordered_key(dist) << 32) | (unsigned)code;
}

__device__ __forceinline__ void finalize_code(const EncArgs& a, int h, int v, unsigned long long packed) {
  const int code = (int)(packed & 0xffffffffull);
  const int b = v / a.T, t = a.t_begin + (v - (v / a.T) * a.T);
  const size_t pair = (size_t)b * a.Hkv + h;
  a.codes[pair * a.n_max + t] = (uint16_t)code;
  if (a.hist) atomicAdd(a.hist + pair * a.L + code, 1);
}

// Argmin over codewords [split * tiles_per_split * 128, ...) for 64 vectors.
__global__ __launch_bounds__(256) void encode_argmin_kernel(EncArgs a) {
  extern __shared__ __align__(16) float smem[];
  float* Ct = smem;
  float* Vt = smem + kD * kCS;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int h = blockIdx.y, split = blockIdx.z;
  const int vec0 = blockIdx.x * kTV;

  for (int idx = tid; idx < kTV * kD; idx += 256) {
    const int vv = idx >> 7, d = idx & (kD - 1);
    const int v = vec0 + vv;
    Vt[d * kVS + vv] = (v < a.nvec) ? a.u[((size_t)h * a.nvec + v) * kD + d] : 0.f;
  }

  float best[8];
  int bidx[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    best[i] = INFINITY;
    bidx[i] = 0x7fffffff;
  }
  const int ntile_total = (a.L + kTC - 1) / kTC;
  const int tbeg = split * a.tiles_per_split, tend = min(ntile_total, tbeg + a.tiles_per_split);
  for (int tile = tbeg; tile < tend; ++tile) {
    const int code0 = tile * kTC;
    __syncthreads();  // previous tile's readers done (and Vt visible on the first pass)
    for (int idx = tid; idx < kTC * 16; idx += 256) {
      const int c = idx & (kTC - 1), dc = idx >> 7;
      const int code = code0 + c;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (code < a.L) v = ld_nc_u4(a.codebook + ((size_t)h * a.L + code) * kD + dc * 8);
      float* col = Ct + (dc * 8) * kCS + c;
      col[0 * kCS] = bf_lo(v.x); col[1 * kCS] = bf_hi(v.x);
      col[2 * kCS] = bf_lo(v.y); col[3 * kCS] = bf_hi(v.y);
      col[4 * kCS] = bf_lo(v.z); col[5 * kCS] = bf_hi(v.z);
      col[6 * kCS] = bf_lo(v.w); col[7 * kCS] = bf_hi(v.w);
    }
    __syncthreads();
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 4
    for (int d = 0; d < kD; ++d) {
      const float4 c4 = *reinterpret_cast<const float4*>(Ct + d * kCS + tx * 4);
      const float4 v0 = *reinterpret_cast<const float4*>(Vt + d * kVS + ty * 8);
      const float4 v1 = *reinterpret_cast<const float4*>(Vt + d * kVS + ty * 8 + 4);
      const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
      const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(vv[i], cc[j], acc[i][j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int code = code0 + tx * 4 + j;
      if (code < a.L) {
        const float n = a.nrm[(size_t)h * a.L + code];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float dist = fmaf(-2.f, acc[i][j], n);
          if (dist < best[i]) {  // codes visited in increasing order: strict < keeps the lowest
            best[i] = dist;
            bidx[i] = code;
          }
        }
      }
    }
  }
  // lexicographic (dist, code) minimum across the 32 lanes (= codeword groups)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best[i], off);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx[i], off);
      if (ob < best[i] || (ob == best[i] && oi < bidx[i])) {
        best[i] = ob;
        bidx[i] = oi;
      }
    }
  }
  const bool single = (gridDim.z == 1);
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int v = vec0 + ty * 8 + i;
      if (v >= a.nvec) break;
      const unsigned long long pk = pack_dist(best[i], bidx[i]);
      if (single) finalize_code(a, h, v, pk);
      else atomicMax(a.slot + (size_t)h * a.nvec + v, ~pk);
    }
  }
  if (single) return;
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(a.counter + (size_t)h * gridDim.x + blockIdx.x, 1u);
    s_last = (prev == gridDim.z - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid < kTV) {
    const int v = vec0 + tid;
    if (v < a.nvec) {
      unsigned long long* sp = a.slot + (size_t)h * a.nvec + v;
      const unsigned long long pk = ~__ldcg(sp);
      finalize_code(a, h, v, pk);
      *sp = 0ull;
    }
  }
  if (tid == 0) a.counter[(size_t)h * gridDim.x + blockIdx.x] = 0u;
}
}  // namespace

cudaError_t launch_prepare(const uint16_t* codebook, const float* H, float* nrm, int Hkv, int L, cudaStream_t st) {
  const int smem = H ? kD * kD * 4 : 0;
  cudaError_t e = cudaFuncSetAttribute(prepare_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kD * kD * 4);
  if (e != cudaSuccess) return e;
  dim3 grid((L + 63) / 64, Hkv);
  prepare_kernel<<<grid, 256, smem, st>>>(codebook, H, nrm, L);
  return cudaGetLastError();
}

cudaError_t launch_encode(const EncArgs& a, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(keyh_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kD * kD * 4);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(encode_argmin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kEncSmem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  dim3 g1((a.nvec + 31) / 32, a.Hkv);
  keyh_kernel<<<g1, 256, a.H ? kD * kD * 4 : 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int ntile_total = (a.L + kTC - 1) / kTC;
  dim3 g2((a.nvec + kTV - 1) / kTV, a.Hkv, (ntile_total + a.tiles_per_split - 1) / a.tiles_per_split);
  encode_argmin_kernel<<<g2, 256, kEncSmem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace a2ats
