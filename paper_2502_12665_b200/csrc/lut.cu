// a1 + a2: WRoPE query rotation and the score table LUT = q~ C^T, folded over
// the GQA group into agg[b, h, l] (Eq. 12, Eq. 21).
//
// lut_umma_kernel: per KV head a dense contraction (M = L codewords, N = B*G
//   queries, K = 2 x 128 for hi and lo) on the 5th-gen tensor cores: one CTA
//   stages a 128-codeword tile with cp.async and computes its query tile
//   q~ = q R_b itself (bf16 hi + lo split, canonical K-major layout); the grid
//   also writes q~ in fp32 and the window table cs[r][m] = (cos, sin)(r f_m)
//   (fp64 angles) for the attention.  One thread issues 16 tcgen05.mma (kind::f16,
//   fp32 accumulator in TMEM), and the epilogue reads its codeword's row
//   (tcgen05.ld), folds the G query heads (max or sum, reading Q10) and writes
//   agg coalesced.  The codebook is exact in bf16 and q~ = hi + lo to ~2^-16, so
//   LUT entries carry fp32-level error (row-relative ~1e-6 << 1e-4).
#include "internal.cuh"
#include "umma.cuh"

namespace a2ats {

namespace {
A2ATS_TL_DECL(g_lut_tl)
A2ATS_PHASE_DECL(g_lut_phase)
constexpr int kTC = 128;  // codewords per CTA (MMA M)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// q~ = q R_b (Eq. 12) for the half-split pairs (m, m+64), m in [m0, m0 + 8): fp32.
__device__ __forceinline__ void rotate8(const LutArgs& a, int qrow, int m0, float y1[8], float y2[8]) {
  const uint4 u1 = ld_nc_u4(a.q + (size_t)qrow * kD + m0);
  const uint4 u2 = ld_nc_u4(a.q + (size_t)qrow * kD + m0 + kHalf);
  const uint32_t w1[4] = {u1.x, u1.y, u1.z, u1.w}, w2[4] = {u2.x, u2.y, u2.z, u2.w};
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float x1 = (e & 1) ? bf_hi(w1[e >> 1]) : bf_lo(w1[e >> 1]);
    const float x2 = (e & 1) ? bf_hi(w2[e >> 1]) : bf_lo(w2[e >> 1]);
    const float2 cs = a.bcs[m0 + e];
    y1[e] = fmaf(x1, cs.x, -x2 * cs.y);
    y2[e] = fmaf(x2, cs.x, x1 * cs.y);
  }
}

__device__ __forceinline__ uint4 pack8(const uint16_t v[8]) {
  return make_uint4(v[0] | (uint32_t(v[1]) << 16), v[2] | (uint32_t(v[3]) << 16), v[4] | (uint32_t(v[5]) << 16),
                    v[6] | (uint32_t(v[7]) << 16));
}

// grid (ceil(L / 128), nvt, Hkv), 128 threads.  Before the dependency wait (inputs
// only): the codeword tile and this CTA's query tile, q~ = q R_b computed here and
// split hi/lo straight into the canonical B layout.  After it: the per-step tables
// the attention reads (q~ fp32, window (cos, sin)), the MMAs and the G-fold epilogue.
template <uint32_t kTmemCols, int G>
__device__ __forceinline__ void lut_body(const LutArgs& a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int NV = a.NV;
  uint8_t* sA = smem;                 // [16 chunks][128 codes][16 B]
  uint8_t* sB = smem + kTC * kD * 2;  // [32 chunks][NV vectors][16 B]: chunks 0..15 hi, 16..31 lo
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.z;
  const int code0 = blockIdx.x * kTC;
  const int vec0 = blockIdx.y * NV;
  const int nvec = a.B * G;

  A2ATS_PHASE(g_lut_phase, 0);
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
  // query tile: vector n = b * G + g <-> q row b * Hq + h * G + g; item = (vector, 8-pair chunk)
#pragma unroll 1
  for (int it = tid; it < NV * 8; it += 128) {
    const int n = it >> 3, c = it & 7, vn = vec0 + n;
    uint16_t h1[8], l1[8], h2[8], l2[8];
    if (vn < nvec) {
      float y1[8], y2[8];
      rotate8(a, (vn / G) * a.Hq + h * G + vn % G, c * 8, y1, y2);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        umma::split_bf16(y1[e], h1[e], l1[e]);
        umma::split_bf16(y2[e], h2[e], l2[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) h1[e] = l1[e] = h2[e] = l2[e] = 0;
    }
    *reinterpret_cast<uint4*>(sB + ((c)*NV + n) * 16) = pack8(h1);        // hi, elements 0..63
    *reinterpret_cast<uint4*>(sB + ((c + 8) * NV + n) * 16) = pack8(h2);  // hi, elements 64..127
    *reinterpret_cast<uint4*>(sB + ((c + 16) * NV + n) * 16) = pack8(l1); // lo
    *reinterpret_cast<uint4*>(sB + ((c + 24) * NV + n) * 16) = pack8(l2);
  }
  A2ATS_PHASE(g_lut_phase, 1);
  pdl_wait();  // the previous step's attention reads qrot / cs; select reads agg
  pdl_trigger();
  if (blockIdx.x == 0) {  // q~ fp32 for the attention (bridge rows), this CTA's vectors
#pragma unroll 1
    for (int it = tid; it < NV * 8; it += 128) {
      const int n = it >> 3, c = it & 7, vn = vec0 + n;
      if (vn >= nvec) continue;
      const int qrow = (vn / G) * a.Hq + h * G + vn % G;
      float y1[8], y2[8];
      rotate8(a, qrow, c * 8, y1, y2);
      float4* dst = reinterpret_cast<float4*>(a.qrot + (size_t)qrow * kD + c * 8);
      dst[0] = make_float4(y1[0], y1[1], y1[2], y1[3]);
      dst[1] = make_float4(y1[4], y1[5], y1[6], y1[7]);
      dst += kHalf / 4;
      dst[0] = make_float4(y2[0], y2[1], y2[2], y2[3]);
      dst[1] = make_float4(y2[4], y2[5], y2[6], y2[7]);
    }
  }
  {  // window relative-rotation table cs[r][m] = (cos, sin)(r f_m) from fp64 angles, spread over the grid
    const int ncta = gridDim.x * gridDim.y * gridDim.z;
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll 1
    for (int i = cta * 128 + tid; i < a.window * kHalf; i += ncta * 128) {
      double sn, cn;
      sincos((double)(i >> 6) * a.rt.inv_freq[i & (kHalf - 1)], &sn, &cn);
      a.cs[i] = make_float2((float)cn, (float)sn);
    }
  }
  cp_async_wait<0>();
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  A2ATS_PHASE(g_lut_phase, 2);
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
  A2ATS_PHASE(g_lut_phase, 3);

  // epilogue: thread <-> codeword row code0 + 32*warp + lane
  const int code = code0 + warp * 32 + lane;
  const int nv_here = min(NV, nvec - vec0);
  const bool sum = (a.group_reduce == A2ATS_GROUP_SUM);
  // rolled over 16-column blocks: this code runs once per CTA, so its size (I-cache
  // misses) costs more than the TMEM load latency it would hide when unrolled
#pragma unroll 1
  for (int col0 = 0; col0 < nv_here; col0 += 16) {
    uint32_t r[16];
    umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + col0, r);
    umma::tmem_wait_ld();
    if (code < a.L) {
      if (a.lut_full) {
#pragma unroll 1
        for (int i = 0; i < 16 && vec0 + col0 + i < nvec; ++i) {
          const int vn = vec0 + col0 + i, b = vn / G, g = vn - b * G;
          float xi = 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j) xi = (j == i) ? __uint_as_float(r[j]) : xi;
          a.lut_full[((size_t)b * a.Hq + h * G + g) * a.L + code] = xi;
        }
      }
#pragma unroll
      for (int bb = 0; bb < 16 / G; ++bb) {  // G divides 16, vec0 + col0 is a multiple of G
        const int n0 = vec0 + col0 + bb * G;
        if (n0 < nvec) {
          float v = __uint_as_float(r[bb * G]);
#pragma unroll
          for (int g = 1; g < G; ++g) {
            const float x = __uint_as_float(r[bb * G + g]);
            v = sum ? v + x : fmaxf(v, x);
          }
          a.agg[((size_t)(n0 / G) * a.Hkv + h) * a.L + code] = v;
        }
      }
    }
  }
  A2ATS_PHASE(g_lut_phase, 4);
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<kTmemCols>(tmem);
}

template <uint32_t kTmemCols, int G>
__global__ __launch_bounds__(128, 1) void lut_umma_kernel(LutArgs a) {
  A2ATS_TL(g_lut_tl, 0);
  lut_body<kTmemCols, G>(a);
  A2ATS_TL(g_lut_tl, 1);
}

// Debug output: scores[b, hq, t] = LUT[b, hq, codes[b, h, t]] for t < n_ctx (Eq. 21).
__global__ void scores_kernel(const float* __restrict__ lut_full, const uint16_t* __restrict__ codes,
                              float* __restrict__ scores, int Hq, int Hkv, int G, int L, int n_max, int n_ctx) {
  pdl_wait();
  pdl_trigger();
  const int bq = blockIdx.y;
  const int b = bq / Hq, hq = bq - (bq / Hq) * Hq, h = hq / G;
  const float* lrow = lut_full + (size_t)bq * L;
  const uint16_t* crow = codes + ((size_t)b * Hkv + h) * n_max;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_ctx; t += gridDim.x * blockDim.x)
    scores[(size_t)bq * n_ctx + t] = lrow[crow[t]];
}

template <uint32_t kCols, int G>
cudaError_t launch_lut_t(const LutArgs& a, cudaStream_t st) {
  const int smem = kTC * kD * 2 + a.NV * 2 * kD * 2;
  static int smem_set = -1;
  if (smem_set < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(lut_umma_kernel<kCols, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  dim3 grid((a.L + kTC - 1) / kTC, a.nvt, a.Hkv);
  return launch_pdl(lut_umma_kernel<kCols, G>, grid, dim3(128), smem, st, a);
}

template <int G>
cudaError_t launch_lut_g(const LutArgs& a, cudaStream_t st) {
  if (a.NV <= 32) return launch_lut_t<32, G>(a, st);
  if (a.NV <= 64) return launch_lut_t<64, G>(a, st);
  if (a.NV <= 128) return launch_lut_t<128, G>(a, st);
  return launch_lut_t<256, G>(a, st);
}
}  // namespace

int lut_tile_nv(int nvec) { return nvec >= 256 ? 256 : ((nvec + 15) / 16) * 16; }  // MMA N: multiple of 16

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
  return launch_pdl(scores_kernel, grid, dim3(256), 0, st, lut_full, codes, scores, Hq, Hkv, G, L, n_max, n_ctx);
}

}  // namespace a2ats

A2ATS_PHASE_EXPORT(a2ats_debug_lut_phases, a2ats::g_lut_phase)

A2ATS_TL_EXPORT(a2ats_debug_lut_timeline, a2ats::g_lut_tl)
