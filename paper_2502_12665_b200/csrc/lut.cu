// a1 + a2: WRoPE query rotation and the score table LUT = q~ C^T, folded over
// the GQA group into agg[b, h, l] (Eq. 12, Eq. 21).
//
// Per KV head this is a dense contraction (M = L codewords, N = B*G queries,
// K = d) run on the 5th-gen tensor cores: one CTA computes a 128-codeword x
// N-query tile with tcgen05.mma (kind::f16, fp32 accumulator in TMEM).
// Precision: the codebook is exact in bf16; q~ (fp32, from fp64 angles) is
// split q~ = hi + lo into two bf16 halves and both are accumulated into the
// same TMEM accumulator (K = 2 x 128), so LUT entries carry ~2^-16 relative
// error (row-relative error ~1e-6 << 1e-4, SURVEY §8c probe).
// The epilogue reads the accumulator row of its codeword (tcgen05.ld), folds
// the G query heads (max or sum, reading Q10) and writes agg coalesced.
#include "internal.cuh"
#include "umma.cuh"

namespace a2ats {

namespace {
constexpr int kTC = 128;  // codewords per CTA (MMA M)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <uint32_t kTmemCols, int G>
__global__ __launch_bounds__(128, 1) void lut_umma_kernel(LutArgs a, int NV) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                // [16 chunks][128 codes][16 B]
  uint8_t* sB = smem + kTC * kD * 2; // [32 chunks][NV vectors][16 B]: chunks 0..15 hi, 16..31 lo
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.z;
  const int code0 = blockIdx.x * kTC;
  const int vec0 = blockIdx.y * NV;
  const int nvec = a.B * G;
  const float2* bcs = a.bcs;

  if (warp == 0) umma::tmem_alloc<kTmemCols>(&tslot);
  if (tid == 0) {
    umma::mbar_init(&mbar, 1);
    umma::mbar_fence_init();
  }

  // codeword tile -> canonical K-major layout (cp.async, 16 B per piece)
  for (int idx = tid; idx < kTC * 16; idx += 128) {
    const int r = idx >> 4, c = idx & 15;
    uint8_t* dst = sA + (c * kTC + r) * 16;
    if (code0 + r < a.L) cp_async16(dst, a.codebook + ((size_t)h * a.L + code0 + r) * kD + c * 8);
    else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
  }
  cp_async_commit();

  // window relative-rotation table cs[r][m] = (cos, sin)(r f_m) from fp64 angles,
  // one row per CTA (linear CTA index r < w)
  const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int nlin = gridDim.x * gridDim.y * gridDim.z;
  for (int r = lin; r < a.window; r += nlin) {
    if (tid < kHalf) {
      double s, c;
      sincos((double)r * a.rt.inv_freq[tid], &s, &c);
      a.cs[r * kHalf + tid] = make_float2((float)c, (float)s);
    }
  }
  // query tile: q~ = q R_b (Eq. 12), half-split pairs (m, m+64); hi/lo bf16 split
  for (int idx = tid; idx < NV * 8; idx += 128) {
    const int n = idx % NV, c = idx / NV;  // chunk c pairs with chunk c+8 (elements m, m+64)
    const int vn = vec0 + n;
    uint16_t h1[8], l1[8], h2[8], l2[8];
    if (vn < nvec) {
      const int b = vn / G, g = vn - b * G;
      const size_t qoff = ((size_t)b * a.Hq + h * G + g) * kD;
      const uint4 x1v = ld_nc_u4(a.q + qoff + c * 8);
      const uint4 x2v = ld_nc_u4(a.q + qoff + kHalf + c * 8);
      const uint32_t w1[4] = {x1v.x, x1v.y, x1v.z, x1v.w}, w2[4] = {x2v.x, x2v.y, x2v.z, x2v.w};
      float y1[8], y2[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float x1 = (i & 1) ? bf_hi(w1[i >> 1]) : bf_lo(w1[i >> 1]);
        const float x2 = (i & 1) ? bf_hi(w2[i >> 1]) : bf_lo(w2[i >> 1]);
        const float2 cs = bcs[c * 8 + i];
        y1[i] = fmaf(x1, cs.x, -x2 * cs.y);
        y2[i] = fmaf(x2, cs.x, x1 * cs.y);
        umma::split_bf16(y1[i], h1[i], l1[i]);
        umma::split_bf16(y2[i], h2[i], l2[i]);
      }
      if (blockIdx.x == 0) {
        float4* q1 = reinterpret_cast<float4*>(a.qrot + qoff + c * 8);
        float4* q2 = reinterpret_cast<float4*>(a.qrot + qoff + kHalf + c * 8);
        q1[0] = make_float4(y1[0], y1[1], y1[2], y1[3]);
        q1[1] = make_float4(y1[4], y1[5], y1[6], y1[7]);
        q2[0] = make_float4(y2[0], y2[1], y2[2], y2[3]);
        q2[1] = make_float4(y2[4], y2[5], y2[6], y2[7]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) h1[i] = l1[i] = h2[i] = l2[i] = 0;
    }
    auto pack = [](const uint16_t* v) {
      return make_uint4(v[0] | (uint32_t(v[1]) << 16), v[2] | (uint32_t(v[3]) << 16), v[4] | (uint32_t(v[5]) << 16),
                        v[6] | (uint32_t(v[7]) << 16));
    };
    *reinterpret_cast<uint4*>(sB + ((c)*NV + n) * 16) = pack(h1);
    *reinterpret_cast<uint4*>(sB + ((c + 8) * NV + n) * 16) = pack(h2);
    *reinterpret_cast<uint4*>(sB + ((16 + c) * NV + n) * 16) = pack(l1);
    *reinterpret_cast<uint4*>(sB + ((24 + c) * NV + n) * 16) = pack(l2);
  }
  cp_async_wait<0>();
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tslot;

  if (tid == 0) {
    const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
    const uint32_t idesc = umma::idesc_bf16(kTC, NV);
#pragma unroll
    for (int s = 0; s < 16; ++s) {  // K = 256: 8 steps against q~_hi, 8 against q~_lo, same A
      const uint64_t ad = umma::sdesc(aBase + (2 * (s & 7)) * (kTC * 16), kTC * 16, 128);
      const uint64_t bd = umma::sdesc(bBase + (2 * s) * (NV * 16), NV * 16, 128);
      umma::mma_bf16(tmem, ad, bd, idesc, s > 0 ? 1u : 0u);
    }
    umma::commit(&mbar);
  }
  __syncwarp();
  umma::mbar_wait(&mbar, 0);
  umma::fence_after();

  // epilogue: thread <-> codeword row code0 + 32*warp + lane
  const int code = code0 + warp * 32 + lane;
  const int nv_here = min(NV, nvec - vec0);
  for (int cb = 0; cb < nv_here; cb += 64) {
    uint32_t r[4][16];
#pragma unroll
    for (int q = 0; q < 4; ++q)  // up to 4 TMEM loads in flight, then one wait
      if (cb + 16 * q < nv_here) umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + cb + 16 * q, r[q]);
    umma::tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
    const int col0 = cb + 16 * q;
    if (col0 >= nv_here) break;
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __uint_as_float(r[q][i]);
    if (code < a.L) {
      if (a.lut_full) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int vn = vec0 + col0 + i;
          if (vn < nvec) {
            const int b = vn / G, g = vn - b * G;
            a.lut_full[((size_t)b * a.Hq + h * G + g) * a.L + code] = x[i];
          }
        }
      }
      const bool sum = (a.group_reduce == A2ATS_GROUP_SUM);
#pragma unroll
      for (int bb = 0; bb < 16 / G; ++bb) {  // G divides 16, vec0 + col0 is a multiple of G
        const int n0 = vec0 + col0 + bb * G;
        if (n0 < nvec) {
          float v = x[bb * G];
#pragma unroll
          for (int g = 1; g < G; ++g) v = sum ? v + x[bb * G + g] : fmaxf(v, x[bb * G + g]);
          a.agg[((size_t)(n0 / G) * a.Hkv + h) * a.L + code] = v;
        }
      }
    }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<kTmemCols>(tmem);
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

template <uint32_t kCols, int G>
cudaError_t launch_lut_t(const LutArgs& a, int NV, cudaStream_t st) {
  const int smem = kTC * kD * 2 + NV * 2 * kD * 2;
  static int smem_set = -1;
  if (smem_set < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(lut_umma_kernel<kCols, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  dim3 grid((a.L + kTC - 1) / kTC, (a.B * G + NV - 1) / NV, a.Hkv);
  lut_umma_kernel<kCols, G><<<grid, 128, smem, st>>>(a, NV);
  return cudaGetLastError();
}

template <int G>
cudaError_t launch_lut_g(const LutArgs& a, cudaStream_t st) {
  const int nvec = a.B * G;
  const int NV = nvec >= 256 ? 256 : ((nvec + 15) / 16) * 16;  // MMA N: multiple of 16, <= 256
  if (NV <= 32) return launch_lut_t<32, G>(a, NV, st);
  if (NV <= 64) return launch_lut_t<64, G>(a, NV, st);
  if (NV <= 128) return launch_lut_t<128, G>(a, NV, st);
  return launch_lut_t<256, G>(a, NV, st);
}
}  // namespace

cudaError_t launch_lut(const LutArgs& a, cudaStream_t st) {
  switch (a.G) {
    case 1: return launch_lut_g<1>(a, st);
    case 2: return launch_lut_g<2>(a, st);
    case 4: return launch_lut_g<4>(a, st);
    default: return launch_lut_g<8>(a, st);
  }
}

cudaError_t launch_scores(const float* lut_full, const uint16_t* codes, float* scores, int B, int Hq, int Hkv,
                          int G, int L, int n_max, int n_ctx, cudaStream_t st) {
  dim3 grid((n_ctx + 1023) / 1024, B * Hq);
  scores_kernel<<<grid, 256, 0, st>>>(lut_full, codes, scores, Hq, Hkv, G, L, n_max, n_ctx);
  return cudaGetLastError();
}

}  // namespace a2ats
