// a1 + a2: WRoPE query rotation and the score table LUT = q~ C^T, folded over
// the GQA group into agg[b, h, l] (Eq. 12, Eq. 21).
//
// lut_umma_kernel: per KV head a dense contraction (M = L codewords, N = B*G
//   queries, K = 2 x 128 for hi and lo) on the 5th-gen tensor cores: one CTA
//   stages a 128-codeword tile with cp.async and computes its query tile
//   q~ = q R_b itself (bf16 hi + lo split, canonical K-major layout); the grid
//   also writes the window table cs[r][m] = (cos, sin)(r f_m) (fp64 angles) for
//   the attention.  One thread issues 16 tcgen05.mma (kind::f16,
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

__device__ __forceinline__ uint4 pack8(const uint16_t v[8]) {
  return make_uint4(v[0] | (uint32_t(v[1]) << 16), v[2] | (uint32_t(v[3]) << 16), v[4] | (uint32_t(v[5]) << 16),
                    v[6] | (uint32_t(v[7]) << 16));
}

// grid (ceil(L / 128), nvt, Hkv), 128 threads.  Before the dependency wait (inputs
// only): the codeword tile and this CTA's query tile, q~ = q R_b computed here and
// split hi/lo straight into the canonical B layout.  After it: the window (cos, sin)
// table the attention reads, the MMAs and the G-fold epilogue.
template <uint32_t kTmemCols, int G>
__device__ __forceinline__ void lut_body(const CUtensorMap& tmA, const LutArgs& a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NV = a.NV;
  uint8_t* sA = smem;                 // 2 x [128 codes][128 B] SW128 K slabs (TMA)
  uint8_t* sB = smem + kTC * kD * 2;  // [32 chunks][NV vectors][16 B]: chunks 0..15 hi, 16..31 lo
  __shared__ uint64_t mbar, tbar;
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
    umma::mbar_init(&tbar, 1);
    umma::mbar_fence_init();
    // codeword tile (rows h*L + code0 .., 128 x 128 bf16) by TMA into two SW128 K slabs;
    // rows past the head belong to the next head (or are zero-filled): never used
    umma::mbar_expect_tx(&tbar, kTC * kD * 2);
    umma::tma_load_2d(sA, &tmA, 0, h * a.L + code0, &tbar);
    umma::tma_load_2d(sA + kTC * 128, &tmA, 64, h * a.L + code0, &tbar);
  }
  __shared__ float2 sbcs[kHalf];  // bridge (cos, sin): smem, not divergent parameter loads
  if (tid < kHalf) sbcs[tid] = a.bcs[tid];
  __syncthreads();
  // query tile: vector n = b * G + g <-> q row b * Hq + h * G + g; item = (vector, 8-pair chunk).
  // All q loads of a pass are issued before any is used (the loop is latency-bound).
  constexpr int kIt = 4;
#pragma unroll 1
  for (int base = 0; base < NV * 8; base += 128 * kIt) {
    uint4 u1[kIt], u2[kIt];
#pragma unroll
    for (int j = 0; j < kIt; ++j) {
      const int it = base + j * 128 + tid, vn = vec0 + (it >> 3);
      u1[j] = u2[j] = make_uint4(0, 0, 0, 0);
      if (it < NV * 8 && vn < nvec) {
        const uint16_t* qp = a.q + (size_t)((vn / G) * a.Hq + h * G + vn % G) * kD + (it & 7) * 8;
        u1[j] = ld_nc_u4(qp);
        u2[j] = ld_nc_u4(qp + kHalf);
      }
    }
#pragma unroll
    for (int j = 0; j < kIt; ++j) {
      const int it = base + j * 128 + tid;
      if (it >= NV * 8) break;
      const int n = it >> 3, c = it & 7;
      const uint32_t w1[4] = {u1[j].x, u1[j].y, u1[j].z, u1[j].w}, w2[4] = {u2[j].x, u2[j].y, u2[j].z, u2[j].w};
      uint16_t h1[8], l1[8], h2[8], l2[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {  // q~ = q R_b (Eq. 12), half-split pair (m, m+64); zero rows stay zero
        const float x1 = (e & 1) ? bf_hi(w1[e >> 1]) : bf_lo(w1[e >> 1]);
        const float x2 = (e & 1) ? bf_hi(w2[e >> 1]) : bf_lo(w2[e >> 1]);
        const float2 cs = sbcs[c * 8 + e];
        umma::split_bf16(fmaf(x1, cs.x, -x2 * cs.y), h1[e], l1[e]);
        umma::split_bf16(fmaf(x2, cs.x, x1 * cs.y), h2[e], l2[e]);
      }
      *reinterpret_cast<uint4*>(sB + ((c)*NV + n) * 16) = pack8(h1);        // hi, elements 0..63
      *reinterpret_cast<uint4*>(sB + ((c + 8) * NV + n) * 16) = pack8(h2);  // hi, elements 64..127
      *reinterpret_cast<uint4*>(sB + ((c + 16) * NV + n) * 16) = pack8(l1); // lo
      *reinterpret_cast<uint4*>(sB + ((c + 24) * NV + n) * 16) = pack8(l2);
    }
  }
  A2ATS_PHASE(g_lut_phase, 1);
  pdl_wait();  // the previous step's attention reads cs; its select reads agg
  pdl_trigger();
  if (tid >= 32) {  // window table cs[r][m] = (cos, sin)(r f_m) from fp64 angles, spread over the grid
    const int ncta = gridDim.x * gridDim.y * gridDim.z;
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll 1
    for (int i = cta * 96 + tid - 32; i < a.window * kHalf; i += ncta * 96) {
      double sn, cn;
      sincos((double)(i >> 6) * a.rt.inv_freq[i & (kHalf - 1)], &sn, &cn);
      a.cs[i] = make_float2((float)cn, (float)sn);
    }
  }
  umma::fence_proxy_async();  // sB (generic-proxy writes) -> tensor core
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  A2ATS_PHASE(g_lut_phase, 2);
  const uint32_t tmem = tslot;

  if (tid == 0) {
    umma::mbar_wait(&tbar, 0);  // codeword tile landed
    const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
    const uint32_t idesc = umma::idesc_bf16(kTC, NV);
#pragma unroll
    for (int s = 0; s < 16; ++s) {  // K = 256: 8 steps against q~_hi, 8 against q~_lo, same A
      const int kk = s & 7;
      const uint64_t ad = umma::sdesc_sw128(aBase + (kk >> 2) * (kTC * 128) + (kk & 3) * 32);
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
__global__ __launch_bounds__(128, 1) void lut_umma_kernel(const __grid_constant__ CUtensorMap tmA, LutArgs a) {
  A2ATS_TL(g_lut_tl, 0);
  lut_body<kTmemCols, G>(tmA, a);
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
cudaError_t launch_lut_t(const LutArgs& a, const CUtensorMap& tm, cudaStream_t st) {
  const int smem = 1024 + kTC * kD * 2 + a.NV * 2 * kD * 2;  // + alignment slack for the SW128 slabs
  static int smem_set = -1;
  if (smem_set < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(lut_umma_kernel<kCols, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  dim3 grid((a.L + kTC - 1) / kTC, a.nvt, a.Hkv);
  return launch_pdl(lut_umma_kernel<kCols, G>, grid, dim3(128), smem, st, tm, a);
}

template <int G>
cudaError_t launch_lut_g(const LutArgs& a, const CUtensorMap& tm, cudaStream_t st) {
  if (a.NV <= 32) return launch_lut_t<32, G>(a, tm, st);
  if (a.NV <= 64) return launch_lut_t<64, G>(a, tm, st);
  if (a.NV <= 128) return launch_lut_t<128, G>(a, tm, st);
  return launch_lut_t<256, G>(a, tm, st);
}
}  // namespace

int lut_tile_nv(int nvec) { return nvec >= 256 ? 256 : ((nvec + 15) / 16) * 16; }  // MMA N: multiple of 16

cudaError_t launch_lut(const LutArgs& a, const CUtensorMap& tm, cudaStream_t st) {
  switch (a.G) {
    case 1: return launch_lut_g<1>(a, tm, st);
    case 2: return launch_lut_g<2>(a, tm, st);
    case 4: return launch_lut_g<4>(a, tm, st);
    default: return launch_lut_g<8>(a, tm, st);
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
