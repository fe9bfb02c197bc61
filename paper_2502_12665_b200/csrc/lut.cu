// a1 + a2: WRoPE query rotation and the score table LUT = q~ C^T, folded over
// the GQA group into agg[b, h, l] (Eq. 12, Eq. 21).
//
// qprep_kernel: q~ = q R_b once per query vector (fp32, for the attention) and
//   its bf16 hi + lo split laid out as the tcgen05 B operand of its KV head; the
//   window relative-rotation table cs[r][m] = (cos, sin)(r f_m) from fp64 angles.
// lut_umma_kernel: per KV head a dense contraction (M = L codewords, N = B*G
//   queries, K = 2 x 128 for hi and lo) on the 5th-gen tensor cores: one CTA
//   stages a 128-codeword tile and the head's query tile with cp.async in the
//   canonical K-major layout, one thread issues 16 tcgen05.mma (kind::f16,
//   fp32 accumulator in TMEM), and the epilogue reads its codeword's row
//   (tcgen05.ld), folds the G query heads (max or sum, reading Q10) and writes
//   agg coalesced.  The codebook is exact in bf16 and q~ = hi + lo to ~2^-16, so
//   LUT entries carry fp32-level error (row-relative ~1e-6 << 1e-4).
#include "internal.cuh"
#include "umma.cuh"

namespace a2ats {

namespace {
A2ATS_PHASE_DECL(g_lut_phase)
constexpr int kTC = 128;  // codewords per CTA (MMA M)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// grid.x = max(B*Hq, window); 64 threads = the 64 rotation pairs (m, m+64).
__global__ __launch_bounds__(64) void qprep_kernel(LutArgs a) {
  const int m = threadIdx.x;
  const int blk = blockIdx.x;
  if (blk < a.window) {  // window table row r = blk
    double s, c;
    sincos((double)blk * a.rt.inv_freq[m], &s, &c);
    a.cs[blk * kHalf + m] = make_float2((float)c, (float)s);
  }
  if (blk < a.B * a.Hq) {
    const int b = blk / a.Hq, hq = blk - b * a.Hq, h = hq / a.G, g = hq - h * a.G;
    const int n = b * a.G + g, vt = n / a.NV, nr = n - vt * a.NV;
    const size_t qoff = (size_t)blk * kD;
    const float x1 = bf_u16(a.q[qoff + m]), x2 = bf_u16(a.q[qoff + m + kHalf]);
    const float2 cs = a.bcs[m];
    const float y1 = fmaf(x1, cs.x, -x2 * cs.y);  // q~ = q R_b (Eq. 12), half-split pair (m, m+64)
    const float y2 = fmaf(x2, cs.x, x1 * cs.y);
    a.qrot[qoff + m] = y1;
    a.qrot[qoff + m + kHalf] = y2;
    uint16_t h1, l1, h2, l2;
    umma::split_bf16(y1, h1, l1);
    umma::split_bf16(y2, h2, l2);
    uint16_t* tile = reinterpret_cast<uint16_t*>(a.qB + ((size_t)(h * a.nvt + vt) * 32) * a.NV * 16);
    const int c = m >> 3, e = m & 7;
    tile[((c)*a.NV + nr) * 8 + e] = h1;            // hi, elements 0..63
    tile[((c + 8) * a.NV + nr) * 8 + e] = h2;      // hi, elements 64..127
    tile[((c + 16) * a.NV + nr) * 8 + e] = l1;     // lo
    tile[((c + 24) * a.NV + nr) * 8 + e] = l2;
  }
  pdl_wait();  // inputs only above; wait for transitivity of the dependency chain
  pdl_trigger();
}

template <uint32_t kTmemCols, int G>
__global__ __launch_bounds__(128, 1) void lut_umma_kernel(LutArgs a) {
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
  // codeword tile -> canonical K-major layout (cp.async, 16 B per piece); a step input
  for (int idx = tid; idx < kTC * 16; idx += 128) {
    const int r = idx >> 4, c = idx & 15;
    uint8_t* dst = sA + (c * kTC + r) * 16;
    if (code0 + r < a.L) cp_async16(dst, a.codebook + ((size_t)h * a.L + code0 + r) * kD + c * 8);
    else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
  }
  cp_async_commit();
  A2ATS_PHASE(g_lut_phase, 1);
  pdl_wait();  // the query tile comes from qprep_kernel
  pdl_trigger();
  {
    const uint8_t* src = a.qB + ((size_t)(h * a.nvt + blockIdx.y) * 32) * NV * 16;
    for (int i = tid; i < 32 * NV; i += 128) cp_async16(sB + i * 16, src + (size_t)i * 16);
    cp_async_commit();
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
  for (int cb = 0; cb < nv_here; cb += 64) {
    uint32_t r[4][16];
#pragma unroll
    for (int q = 0; q < 4; ++q)  // up to 4 TMEM loads in flight, then one wait
      if (cb + 16 * q < nv_here) umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + cb + 16 * q, r[q]);
    umma::tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int col0 = cb + 16 * q;
      if (col0 >= nv_here || code >= a.L) break;
      float x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = __uint_as_float(r[q][i]);
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
  A2ATS_PHASE(g_lut_phase, 4);
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<kTmemCols>(tmem);
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
  const int grid = max(a.B * a.Hq, a.window);
  cudaError_t e = launch_pdl(qprep_kernel, dim3(grid), dim3(kHalf), 0, st, a);
  if (e != cudaSuccess) return e;
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
