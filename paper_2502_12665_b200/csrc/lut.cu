// a1 + a2: WRoPE query rotation and the score table LUT = q~ C^T, folded over
// the GQA group into agg[b, h, l] (Eq. 12, Eq. 21).
//
// v1 kernel: fp32 FMA GEMM tile (128 codewords x 64 query vectors per CTA,
// 4x8 register micro-tile per thread).  The bf16 codebook is converted exactly
// to fp32 in shared memory; q~ is fp32 from fp64 angles, so every LUT entry is
// an fp32-accumulated dot product (row-relative error ~1e-7 << 1e-4).
#include "internal.cuh"

namespace a2ats {

namespace {
constexpr int kTC = 128;          // codewords per CTA
constexpr int kTV = 64;           // query vectors per CTA
constexpr int kCS = kTC + 4;      // C^T row stride (floats)
constexpr int kVS = kTV + 4;      // Q^T row stride (floats)
constexpr int kLutSmem = (kD * kCS + kD * kVS) * 4;

__global__ __launch_bounds__(256) void lut_fma_kernel(LutArgs a) {
  extern __shared__ __align__(16) float smem[];
  float* Ct = smem;               // [128 d][kCS]  codeword tile, transposed
  float* Vt = smem + kD * kCS;    // [128 d][kVS]  rotated queries, transposed
  __shared__ float2 bcs[kHalf];   // (cos, sin)(b f_m)

  const int tid = threadIdx.x;
  const int h = blockIdx.z;
  const int code0 = blockIdx.x * kTC;
  const int vec0 = blockIdx.y * kTV;
  const int nvec = a.B * a.G;

  // Window relative-rotation table cs[r][m] = (cos, sin)(r f_m), r < w, from fp64
  // angles; spread over the first CTAs (row r by linear CTA r).
  const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int nlin = gridDim.x * gridDim.y * gridDim.z;
  for (int r = lin; r < a.window; r += nlin) {
    if (tid < kHalf) {
      double s, c;
      sincos((double)r * a.rt.inv_freq[tid], &s, &c);
      a.cs[r * kHalf + tid] = make_float2((float)c, (float)s);
    }
  }
  if (tid < kHalf) {
    double s, c;
    sincos((double)a.bridge * a.rt.inv_freq[tid], &s, &c);
    bcs[tid] = make_float2((float)c, (float)s);
  }

  // Codeword tile -> C^T (exact bf16 -> fp32).
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
  __syncthreads();  // bcs visible

  // Query tile: q~ = q R_b (Eq. 12), half-split pairs (m, m+64).
  for (int idx = tid; idx < kTV * kHalf; idx += 256) {
    const int m = idx & (kHalf - 1), vv = idx >> 6;
    const int n = vec0 + vv;
    float x1 = 0.f, x2 = 0.f;
    size_t qoff = 0;
    if (n < nvec) {
      const int b = n / a.G, g = n - (n / a.G) * a.G;
      qoff = ((size_t)b * a.Hq + h * a.G + g) * kD;
      x1 = bf_u16(a.q[qoff + m]);
      x2 = bf_u16(a.q[qoff + m + kHalf]);
    }
    const float2 cs = bcs[m];
    const float y1 = fmaf(x1, cs.x, -x2 * cs.y);
    const float y2 = fmaf(x2, cs.x, x1 * cs.y);
    Vt[m * kVS + vv] = y1;
    Vt[(m + kHalf) * kVS + vv] = y2;
    if (blockIdx.x == 0 && n < nvec) {
      a.qrot[qoff + m] = y1;
      a.qrot[qoff + m + kHalf] = y2;
    }
  }
  __syncthreads();

  const int tx = tid & 31, ty = tid >> 5;
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

  const int cbase = code0 + tx * 4;
  if (a.lut_full) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int n = vec0 + ty * 8 + i;
      if (n >= nvec) break;
      const int b = n / a.G, g = n - (n / a.G) * a.G;
      float* dst = a.lut_full + ((size_t)b * a.Hq + h * a.G + g) * a.L;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (cbase + j < a.L) dst[cbase + j] = acc[i][j];
    }
  }
  // Fold the G query heads of each batch element (G divides 8; vec0 % G == 0).
  const int nb = 8 / a.G;
  for (int bb = 0; bb < nb; ++bb) {
    const int n0 = vec0 + ty * 8 + bb * a.G;
    if (n0 >= nvec) break;
    const int b = n0 / a.G;
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float x = acc[bb * a.G][j];
      for (int g = 1; g < a.G; ++g) {
        const float y = acc[bb * a.G + g][j];
        x = (a.group_reduce == A2ATS_GROUP_SUM) ? x + y : fmaxf(x, y);
      }
      r[j] = x;
    }
    float* dst = a.agg + ((size_t)b * a.Hkv + h) * a.L;
    if (cbase + 3 < a.L && (a.L & 3) == 0) {
      *reinterpret_cast<float4*>(dst + cbase) = make_float4(r[0], r[1], r[2], r[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (cbase + j < a.L) dst[cbase + j] = r[j];
    }
  }
}

// Debug output: scores[b, hq, t] = LUT[b, hq, codes[b, h, t]] for t < n_ctx (Eq. 21).
__global__ void scores_kernel(const float* __restrict__ lut_full, const uint16_t* __restrict__ codes,
                              float* __restrict__ scores, int Hq, int Hkv, int G, int L, int n_max, int n_ctx) {
  const int bq = blockIdx.y;
  const int b = bq / Hq, hq = bq - (bq / Hq) * Hq, h = hq / G;
  const float* lrow = lut_full + (size_t)bq * L;
  const uint16_t* crow = codes + ((size_t)b * Hkv + h) * n_max;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_ctx; t += gridDim.x * blockDim.x)
    scores[(size_t)bq * n_ctx + t] = lrow[crow[t]];
}
}  // namespace

cudaError_t launch_lut(const LutArgs& a, cudaStream_t st) {
  static bool attr_done = false;  // per process; single-device use is the norm
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(lut_fma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLutSmem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  dim3 grid((a.L + kTC - 1) / kTC, (a.B * a.G + kTV - 1) / kTV, a.Hkv);
  lut_fma_kernel<<<grid, 256, kLutSmem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_scores(const float* lut_full, const uint16_t* codes, float* scores, int B, int Hq, int Hkv,
                          int G, int L, int n_max, int n_ctx, cudaStream_t st) {
  dim3 grid((n_ctx + 1023) / 1024, B * Hq);
  scores_kernel<<<grid, 256, 0, st>>>(lut_full, codes, scores, Hq, Hkv, G, L, n_max, n_ctx);
  return cudaGetLastError();
}

}  // namespace a2ats
