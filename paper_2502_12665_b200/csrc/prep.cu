// The step's first kernel: three independent roles in one launch, so that the
// score table, the new key's code and the window logits are computed concurrently
// (one CTA per tile of one role; every role reads only step inputs before the
// dependency wait).
//
// LUT role (a1 + a2; Eq. 12, Eq. 21): per KV head a dense
//   contraction M = L codewords, N = B*G queries, K = 2 x 128 (q~ hi and lo) on the
//   5th-gen tensor cores.  A CTA loads a 128-codeword tile by TMA (SWIZZLE_128B),
//   computes its query tile q~ = q R_b itself (fp32 from fp64 angles, split into bf16
//   hi + lo in the canonical K-major layout), issues 16 tcgen05.mma into TMEM, and the
//   epilogue folds the G query heads (max or sum, reading Q10) into agg.  The codebook
//   is exact in bf16 and q~ = hi + lo to ~2^-16, so LUT entries carry fp32-level error.
//   The LUT CTAs also write the window table cs[r][m] = (cos, sin)(r f_m) (fp64
//   angles) used by the attention for window rows beyond the precomputed ones.
// Encode role (a0 for the decode step's new keys; Eq. 14, Eq. 20):
//   encode_tile of encode_common.cuh.
// Window role (a5's local rows; Eq. 11): for one (b, KV head) pair, the
//   logits u_j = (q R_{i-j}) . k_j of the first min(w, 64) window tokens, an exact
//   per-row rotation on FP32 cores ((cos, sin)(r f_m) from an fp64 angle at the first
//   row, then fp64 rotations by -f_m per row), base-2 scaled, into wlog.
#include "encode_common.cuh"

namespace a2ats {

namespace {
A2ATS_TL_DECL(g_prep_tl)
A2ATS_PHASE_DECL(g_lut_phase)
constexpr int kTC = 128;  // codewords per LUT CTA (MMA M)

__device__ __forceinline__ uint4 pack8(const uint16_t v[8]) {
  return make_uint4(v[0] | (uint32_t(v[1]) << 16), v[2] | (uint32_t(v[3]) << 16), v[4] | (uint32_t(v[5]) << 16),
                    v[6] | (uint32_t(v[7]) << 16));
}

__host__ __device__ constexpr int lut_tile_smem(int NV) { return kTC * kD * 2 + NV * 2 * kD * 2; }
constexpr int kWinSmem = 32768 + 16384 + 8 * kD * 4;  // cs [64][64] float2, K [64][128] bf16, q [8][128] fp32

// LUT tile i of p.n_lut: (code tile x, vector tile y, head h).  Before the dependency
// wait: codeword tile (TMA) and q~ tile; after: the cs table share, MMAs, G-fold epilogue.
template <int G>
__device__ __forceinline__ void lut_tile(const CUtensorMap& tmA, const PrepArgs& p, int i, uint8_t* smem) {
  const LutArgs& a = p.lut;
  const int NV = a.NV;
  uint8_t* sA = smem;                 // 2 x [128 codes][128 B] SW128 K slabs (TMA)
  uint8_t* sB = smem + kTC * kD * 2;  // [32 chunks][NV vectors][16 B]: chunks 0..15 hi, 16..31 lo
  __shared__ uint64_t mbar, tbar;
  __shared__ uint32_t tslot;
  __shared__ float2 sbcs[kHalf];  // bridge (cos, sin): smem, not divergent parameter loads

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cx_n = (p.lut_tx + p.lut_tpc - 1) / p.lut_tpc;  // CTAs per (vector tile, head)
  const int cx = i % cx_n, y = (i / cx_n) % a.nvt, h = i / (cx_n * a.nvt);
  const int xt0 = cx * p.lut_tpc, xt1 = min(p.lut_tx, xt0 + p.lut_tpc);  // code tiles of this CTA
  const int vec0 = y * NV;
  const int nvec = a.B * G;

  A2ATS_PHASE(g_lut_phase, 0);
  if (warp == 0) umma::tmem_alloc_n(&tslot, p.lut_cols);
  if (tid == 0) {
    umma::mbar_init(&mbar, 1);
    umma::mbar_init(&tbar, 1);
    umma::mbar_fence_init();
    // codeword tile (rows h*L + code0 .., 128 x 128 bf16) by TMA into two SW128 K slabs;
    // rows past the head belong to the next head (or are zero-filled): never used
    umma::mbar_expect_tx(&tbar, kTC * kD * 2);
    umma::tma_load_2d(sA, &tmA, 0, h * a.L + xt0 * kTC, &tbar);
    umma::tma_load_2d(sA + kTC * 128, &tmA, 64, h * a.L + xt0 * kTC, &tbar);
  }
  if (!a.qt && tid < kHalf) sbcs[tid] = a.bcs[tid];  // (precomputed q~ tiles need no rotation here)
  __syncthreads();
  if (!a.qt) {
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
  }
  A2ATS_PHASE(g_lut_phase, 1);
  A2ATS_TL(g_prep_tl, 2);
  pdl_wait();  // the previous step's attention reads cs; its select reads agg
  pdl_trigger();
  A2ATS_TL(g_prep_tl, 3);
  if (a.qt) {  // precomputed q~ tile (qprep_kernel, complete: this CTA passed its dependency wait)
    __shared__ uint64_t qbar;
    if (tid == 0) {
      umma::mbar_init(&qbar, 1);
      umma::mbar_fence_init();
      umma::mbar_expect_tx(&qbar, (uint32_t)NV * 32 * 16);
      umma::bulk_load(sB, a.qt + ((size_t)h * a.nvt + y) * 32 * NV * 8, (uint32_t)NV * 32 * 16, &qbar);
    }
    __syncthreads();
    umma::mbar_wait(&qbar, 0);
  }
  if (!a.qt && tid >= 32) {  // window table cs[r][m] = (cos, sin)(r f_m) from fp64 angles, spread over the LUT CTAs
#pragma unroll 1
    for (int k = i * 96 + tid - 32; k < a.window * kHalf; k += p.n_lut * 96) {
      double sn, cn;
      sincos((double)(k >> 6) * a.rt.inv_freq[k & (kHalf - 1)], &sn, &cn);
      a.cs[k] = make_float2((float)cn, (float)sn);
    }
  }
  umma::fence_proxy_async();  // sB (generic-proxy writes) -> tensor core
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  A2ATS_PHASE(g_lut_phase, 2);
  A2ATS_TL(g_prep_tl, 4);
  const uint32_t tmem = tslot;
  const uint32_t idesc = umma::idesc_bf16(kTC, NV);
  const int nv_here = min(NV, nvec - vec0);
  const bool sum = (a.group_reduce == A2ATS_GROUP_SUM);
#pragma unroll 1
  for (int xt = xt0; xt < xt1; ++xt) {  // code tiles one after the other, same q~ tile
    const int it = xt - xt0, code0 = xt * kTC;
    if (tid == 0) {
      umma::mbar_wait(&tbar, it & 1);  // codeword tile landed
      const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
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
    umma::mbar_wait(&mbar, it & 1);
    umma::fence_after();
    if (it == 0) A2ATS_TL(g_prep_tl, 5);
    if (tid == 0 && xt + 1 < xt1) {  // next codeword tile into the (now free) A buffer
      umma::mbar_expect_tx(&tbar, kTC * kD * 2);
      umma::tma_load_2d(sA, &tmA, 0, h * a.L + code0 + kTC, &tbar);
      umma::tma_load_2d(sA + kTC * 128, &tmA, 64, h * a.L + code0 + kTC, &tbar);
    }
    A2ATS_PHASE(g_lut_phase, 3);

    // epilogue: thread <-> codeword row code0 + 32*warp + lane; the G-fold of each group of G
    // columns (one batch element) is stored at agg[b][h][code]: one pointer, one stride
    const int code = code0 + warp * 32 + lane;
    const bool live = code < a.L;
    const size_t bstride = (size_t)a.Hkv * a.L;
    float* aggp = a.agg + ((size_t)(vec0 / G) * a.Hkv + h) * a.L + code;
    auto fold = [&](const uint32_t* r, int col0) {
      if (a.lut_full && live) {
#pragma unroll 1
        for (int ii = 0; ii < 16 && vec0 + col0 + ii < nvec; ++ii) {
          const int vn = vec0 + col0 + ii, b = vn / G, g = vn - b * G;
          float xi = 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j) xi = (j == ii) ? __uint_as_float(r[j]) : xi;
          a.lut_full[((size_t)b * a.Hq + h * G + g) * a.L + code] = xi;
        }
      }
      float* pb = aggp + (size_t)(col0 / G) * bstride;
#pragma unroll
      for (int bb = 0; bb < 16 / G; ++bb) {  // G divides 16, vec0 + col0 is a multiple of G
        float v = __uint_as_float(r[bb * G]);
#pragma unroll
        for (int g = 1; g < G; ++g) {
          const float xg = __uint_as_float(r[bb * G + g]);
          v = sum ? v + xg : fmaxf(v, xg);
        }
        if (live && col0 + bb * G < nv_here) pb[bb * bstride] = v;
      }
    };
    // 32-column blocks, software-pipelined: the next block's TMEM load is in flight while this
    // block is folded and stored (columns past nv_here: allocated, never stored)
    {
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
      uint32_t ra[32], rb[32];
      umma::tmem_ld32(ta, ra);
      umma::tmem_wait_ld();
#pragma unroll 1
      for (int col0 = 0; col0 < nv_here; col0 += 64) {
        const bool nb = col0 + 32 < nv_here;
        if (nb) umma::tmem_ld32(ta + col0 + 32, rb);
        fold(ra, col0);
        fold(ra + 16, col0 + 16);
        if (nb) {
          umma::tmem_wait_ld();
          if (col0 + 64 < nv_here) umma::tmem_ld32(ta + col0 + 64, ra);
          fold(rb, col0 + 32);
          fold(rb + 16, col0 + 48);
          if (col0 + 64 < nv_here) umma::tmem_wait_ld();
        }
      }
    }
    umma::fence_before();
    __syncthreads();  // TMEM read out before the next tile's MMAs
    umma::fence_after();
    if (it == 0) A2ATS_TL(g_prep_tl, 6);
  }
  A2ATS_PHASE(g_lut_phase, 4);
  if (warp == 0) umma::tmem_dealloc_n(tmem, p.lut_cols);
}

// Persistent warp-specialized LUT (a2; wide query tiles with precomputed q~, la.qt): one CTA
// per SM walks a contiguous range of units (head h, vector tile y, 128-codeword tile x), x
// fastest, so consecutive units share the q~ B tile.  Warp 0 produces (codeword tile by TMA,
// B tile by bulk copy when (h, y) changes), warp 1 issues the 16 tcgen05.mma of a unit into one
// of two TMEM accumulators, warps 2..9 drain the other accumulator (8 warps: TMEM lane quarter
// w % 4, column half (w - 2) / 4), fold the G heads and store agg -- so the next unit's codeword
// load and MMAs run under the current unit's epilogue, whose TMEM reads bound the kernel.
constexpr int kLpWarps = 10;  // producer, MMA, 8 epilogue warps
constexpr int kLpStages = 2;  // codeword-tile ring: the next unit's tile loads while this unit's MMAs run
__host__ __device__ constexpr int lut_persist_smem(int NV) {
  return kLpStages * kTC * kD * 2 + NV * 2 * kD * 2 + 1024;
}

template <int G>
// (<= 96 registers: with the LUT CTA's 320 threads, two posting-select CTAs (256 x 64) still fit on
// its SM, so they run their step-input prologue during the LUT)
__global__ __launch_bounds__(kLpWarps * 32, 2) void lut_persist_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                       const LutArgs a, int n_units, int ntx) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + kLpStages * kTC * kD * 2;  // [32 chunks][NV vectors][16 B]
  __shared__ __align__(8) uint64_t a_full[kLpStages], a_empty[kLpStages], b_full, b_empty, t_full[2], t_empty[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NV = a.NV, ncols = (int)umma::tmem_cols_for(NV);
  const int u0 = (int)((long long)blockIdx.x * n_units / gridDim.x);
  const int u1 = (int)((long long)(blockIdx.x + 1) * n_units / gridDim.x);
  auto hy_of = [&](int u) { return u / ntx; };  // (h, y) block index = h * nvt + y
  auto issue_a = [&](int u, int st) {           // codeword tile of unit u into ring stage st
    const int h = hy_of(u) / a.nvt, x = u % ntx;
    uint8_t* d = sA + st * (kTC * kD * 2);
    umma::mbar_expect_tx(&a_full[st], kTC * kD * 2);
    umma::tma_load_2d(d, &tmA, 0, h * a.L + x * kTC, &a_full[st]);
    umma::tma_load_2d(d + kTC * 128, &tmA, 64, h * a.L + x * kTC, &a_full[st]);
  };
  if (tid == 0) {
    for (int st = 0; st < kLpStages; ++st) {
      umma::mbar_init(&a_full[st], 1);
      umma::mbar_init(&a_empty[st], 1);
    }
    umma::mbar_init(&b_full, 1);
    umma::mbar_init(&b_empty, 1);
    for (int j = 0; j < 2; ++j) {
      umma::mbar_init(&t_full[j], 1);
      umma::mbar_init(&t_empty[j], 8);
    }
    umma::mbar_fence_init();
    // the first codeword tiles (step inputs) before the dependency wait
    for (int st = 0; st < kLpStages && u0 + st < u1; ++st) issue_a(u0 + st, st);
  }
  A2ATS_TL(g_prep_tl, 0);
  if (warp == 1) umma::tmem_alloc_n(&tslot, 2 * ncols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tslot;
  // q~ tiles come from qprep_kernel; the previous step's select reads agg.  Dependents may launch
  // now: their pre-wait prologues read only step inputs
  pdl_wait();
  pdl_trigger();
  A2ATS_TL(g_prep_tl, 2);
  if (warp == 0) {
    if (lane == 0) {  // producer
      int nb = 0, cur = -1;
      for (int u = u0, it = 0; u < u1; ++u, ++it) {
        const int hy = hy_of(u), st = it % kLpStages;
        if (it >= kLpStages) {  // (the first kLpStages tiles were issued before the wait)
          umma::mbar_wait(&a_empty[st], ((it - kLpStages) / kLpStages) & 1);  // unit it - S's MMAs done
          issue_a(u, st);
        }
        if (hy != cur) {
          if (nb > 0) umma::mbar_wait(&b_empty, (nb - 1) & 1);
          umma::mbar_expect_tx(&b_full, (uint32_t)NV * 32 * 16);
          umma::bulk_load(sB, a.qt + (size_t)hy * 32 * NV * 8, (uint32_t)NV * 32 * 16, &b_full);
          cur = hy;
          ++nb;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = umma::idesc_bf16(kTC, NV);
      const uint32_t bBase = smem_u32(sB);
      int nb = 0, cur = -1;
      for (int u = u0, it = 0; u < u1; ++u, ++it) {
        const int j = it & 1, hy = hy_of(u), st = it % kLpStages;
        const uint32_t aBase = smem_u32(sA + st * (kTC * kD * 2));
        if (it >= 2) umma::mbar_wait(&t_empty[j], ((it - 2) >> 1) & 1);  // accumulator j drained
        umma::mbar_wait(&a_full[st], (it / kLpStages) & 1);
        if (it == 0) A2ATS_TLX(g_prep_tl, 6);
        if (hy != cur) {
          umma::mbar_wait(&b_full, nb & 1);
          cur = hy;
          ++nb;
        }
        if (it == 0) A2ATS_TLX(g_prep_tl, 7);
        umma::fence_after();
        const uint32_t td = tmem + (uint32_t)(j * ncols);
#pragma unroll
        for (int s = 0; s < 16; ++s) {  // K = 256: 8 steps against q~_hi, 8 against q~_lo, same A
          const int kk = s & 7;
          const uint64_t ad = umma::sdesc_sw128(aBase + (kk >> 2) * (kTC * 128) + (kk & 3) * 32);
          const uint64_t bd = umma::sdesc(bBase + (2 * s) * (NV * 16), NV * 16, 128);
          umma::mma_bf16(td, ad, bd, idesc, s > 0 ? 1u : 0u);
        }
        umma::commit(&a_empty[st]);                             // stage st reusable once these MMAs complete
        if (u + 1 == u1 || hy_of(u + 1) != hy) umma::commit(&b_empty);  // last unit on this B tile
        umma::commit(&t_full[j]);
      }
    }
  } else {  // epilogue: TMEM lane quarter q, columns [half * NV / 2, (half + 1) * NV / 2)
    const int q = warp & 3, half = (warp - 2) >> 2, nvec = a.B * G;
    const bool sum = (a.group_reduce == A2ATS_GROUP_SUM);
    const size_t bstride = (size_t)a.Hkv * a.L;
    if (a.cs_in_lut)  // window table cs[r][m] (fp64 angles) while the first MMA runs
      for (int k = blockIdx.x * 256 + tid - 64; k < a.window * kHalf; k += gridDim.x * 256) {
        double sn, cn;
        sincos((double)(k >> 6) * a.rt.inv_freq[k & (kHalf - 1)], &sn, &cn);
        a.cs[k] = make_float2((float)cn, (float)sn);
      }
    for (int u = u0, it = 0; u < u1; ++u, ++it) {
      const int j = it & 1, hy = hy_of(u), h = hy / a.nvt, y = hy % a.nvt, x = u % ntx;
      const int vec0 = y * NV, nv_here = min(NV, nvec - vec0);
      const int code = x * kTC + q * 32 + lane;
      const bool live = code < a.L;
      float* aggp = a.agg + ((size_t)(vec0 / G) * a.Hkv + h) * a.L + code;
      umma::mbar_wait(&t_full[j], (it >> 1) & 1);
      umma::fence_after();
      if (tid == 64 && it == 0) A2ATS_TLX(g_prep_tl, 3);
      if (tid == 64 && u + 1 == u1) A2ATS_TLX(g_prep_tl, 5);
      const uint32_t ta = tmem + (uint32_t)(j * ncols) + ((uint32_t)(q * 32) << 16);
      auto fold = [&](const uint32_t* r, int col0) {  // 16 columns = 16 / G batch elements
        if (a.lut_full && live) {
#pragma unroll 1
          for (int ii = 0; ii < 16 && col0 + ii < nv_here; ++ii) {
            const int vn = vec0 + col0 + ii, b = vn / G, g = vn - b * G;
            float xi = 0.f;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) xi = (jj == ii) ? __uint_as_float(r[jj]) : xi;
            a.lut_full[((size_t)b * a.Hq + h * G + g) * a.L + code] = xi;
          }
        }
        float* pb = aggp + (size_t)(col0 / G) * bstride;
#pragma unroll
        for (int bb = 0; bb < 16 / G; ++bb) {
          float v = __uint_as_float(r[bb * G]);
#pragma unroll
          for (int g = 1; g < G; ++g) {
            const float xg = __uint_as_float(r[bb * G + g]);
            v = sum ? v + xg : fmaxf(v, xg);
          }
          if (live && col0 + bb * G < nv_here) pb[bb * bstride] = v;
        }
      };
      const int c_lo = half * (NV >> 1), c_hi = min(c_lo + (NV >> 1), nv_here);
      for (int col0 = c_lo; col0 < c_hi; col0 += 32) {
        uint32_t r[32];
        umma::tmem_ld32(ta + col0, r);
        umma::tmem_wait_ld();
        fold(r, col0);
        fold(r + 16, col0 + 16);
      }
      umma::fence_before();
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(&t_empty[j]);
      if (tid == 64 && it == 0) A2ATS_TLX(g_prep_tl, 4);
    }
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (warp == 1) umma::tmem_dealloc_n(tmem, 2 * ncols);
  A2ATS_TL(g_prep_tl, 1);
}

// Window role: pairs [pair0, pair0 + np) (the window rows, hence the rotation table, are
// the same for every pair).  Scratch (16-B chunks XOR-swizzled by row): cs [64][64] float2,
// K rows [64][128] bf16, q (base-2 scaled) [8][128] fp32.
__device__ __forceinline__ void window_tile(const PrepArgs& p, int pair0, int np, uint8_t* smem) {
  const LutArgs& a = p.lut;
  const int tid = threadIdx.x, G = a.G, nw = p.n_wl;
  float4* csS = reinterpret_cast<float4*>(smem);                // [64 rows][32 chunks of 2 (cos, sin)]
  uint4* kS = reinterpret_cast<uint4*>(smem + 32768);           // [64 rows][16 chunks of 8 bf16]
  float* sQ = reinterpret_cast<float*>(smem + 32768 + 16384);   // [8][128]
  {
    const int m = tid & 63, j0 = (tid >> 6) * 32;  // rows [j0, j0 + 32) of pair m
    if (j0 < nw) {
      const double f = a.rt.inv_freq[m];
      double sn, cn, sf, cf;
      sincos((double)(p.n_ctx - 1 - (p.win_lo + j0)) * f, &sn, &cn);  // r = i - t, t = win_lo + row
      sincos(f, &sf, &cf);
      float2* cs2 = reinterpret_cast<float2*>(csS);
#pragma unroll 1
      for (int row = j0; row < min(j0 + 32, nw); ++row) {
        cs2[row * 64 + (((m >> 1) ^ (row & 7)) << 1) + (m & 1)] = make_float2((float)cn, (float)sn);
        const double c2 = cn * cf + sn * sf, s2 = sn * cf - cn * sf;  // r -> r - 1
        cn = c2;
        sn = s2;
      }
    }
  }
  A2ATS_TL(g_prep_tl, 2);
  const int row = tid & 63, hsel = tid >> 6;  // heads hsel, hsel + 2, ...
#pragma unroll 1
  for (int pair = pair0; pair < pair0 + np; ++pair) {
    const int b = pair / a.Hkv, h = pair - b * a.Hkv;
    const uint8_t* kbase = reinterpret_cast<const uint8_t*>(p.kc) + (size_t)pair * p.n_max * 256;
    {  // q of the group's heads, scaled to the base-2 logit domain (one 16-B load per thread)
      const int g = tid >> 4, e0 = (tid & 15) * 8;
      uint4 xq = make_uint4(0, 0, 0, 0);
      if (g < G) xq = ld_nc_u4(a.q + ((size_t)b * a.Hq + h * G + g) * kD + e0);
      const uint32_t w[4] = {xq.x, xq.y, xq.z, xq.w};
      float4* d = reinterpret_cast<float4*>(sQ + g * kD + e0);
      d[0] = make_float4(bf_lo(w[0]) * p.scale_log2, bf_hi(w[0]) * p.scale_log2, bf_lo(w[1]) * p.scale_log2,
                         bf_hi(w[1]) * p.scale_log2);
      d[1] = make_float4(bf_lo(w[2]) * p.scale_log2, bf_hi(w[2]) * p.scale_log2, bf_lo(w[3]) * p.scale_log2,
                         bf_hi(w[3]) * p.scale_log2);
    }
    for (int k = tid; k < nw * 16; k += 128) {
      const int r = k >> 4, c = k & 15;
      kS[r * 16 + (c ^ (r & 7))] = ld_nc_u4(kbase + (size_t)(p.win_lo + r - p.shard_begin) * 256 + c * 16);
    }
    __syncthreads();
    if (pair == pair0) A2ATS_TL(g_prep_tl, 3);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (row < nw) {
#pragma unroll 1
      for (int mb = 0; mb < 8; ++mb) {  // m = 8 mb + i; pairs (m, m + 64)
        const uint4 k1 = kS[row * 16 + (mb ^ (row & 7))];
        const uint4 k2 = kS[row * 16 + ((mb + 8) ^ (row & 7))];
        const uint32_t w1[4] = {k1.x, k1.y, k1.z, k1.w}, w2[4] = {k2.x, k2.y, k2.z, k2.w};
        float4 t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = csS[row * 32 + ((mb * 4 + j) ^ (row & 7))];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
          const int g = hsel + 2 * hh;
          if (g < G) {
            const float* qa = sQ + g * kD + mb * 8;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float ka = (e & 1) ? bf_hi(w1[e >> 1]) : bf_lo(w1[e >> 1]);
              const float kb = (e & 1) ? bf_hi(w2[e >> 1]) : bf_lo(w2[e >> 1]);
              const float cv = (e & 1) ? t[e >> 1].z : t[e >> 1].x, sv = (e & 1) ? t[e >> 1].w : t[e >> 1].y;
              const float q1 = qa[e], q2 = qa[e + kHalf];
              acc[hh] = fmaf(cv, fmaf(q1, ka, q2 * kb), fmaf(sv, fmaf(q1, kb, -q2 * ka), acc[hh]));
            }
          }
        }
      }
    }
    if (pair == pair0) {
      A2ATS_TL(g_prep_tl, 4);
      pdl_wait();  // the previous step's attention reads wlog
      pdl_trigger();
      A2ATS_TL(g_prep_tl, 5);
    }
    if (row < nw) {
#pragma unroll
      for (int hh = 0; hh < 4; ++hh)
        p.wlog[((size_t)pair * kWinPre + row) * 8 + hsel + 2 * hh] = acc[hh];  // heads >= G: 0
    }
    __syncthreads();  // q / K scratch reused by the next pair
  }
  if (np == 0) {
    pdl_wait();
    pdl_trigger();
  }
}

// q~ = q R_b (Eq. 12) split into bf16 hi + lo, in the LUT's canonical K-major B layout:
// tile (h, y) = [32 chunks (0..15 hi, 16..31 lo)][NV vectors][8 bf16]; vectors past B*G are 0.
// Thread <-> (tile, 8-pair chunk c, vector n), n fastest (coalesced 16-B stores).  Also writes
// the window table cs (fp64 angles) that the LUT CTAs write when there is no qprep.
__global__ __launch_bounds__(256) void qprep_kernel(LutArgs a) {
#ifdef A2ATS_PHASES
  if (threadIdx.x == 0) {  // timeline rows 4096.. (tuning builds)
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_prep_tl[4096 + blockIdx.x][0] = t_;
  }
#endif
  // step inputs first (q, the bridge rotation), the q~ tile written after the dependency wait
  __shared__ float2 sbcs[kHalf];  // bridge (cos, sin) in smem: per-lane indices would serialize param loads
  if (threadIdx.x < kHalf) sbcs[threadIdx.x] = a.bcs[threadIdx.x];
  const int NV = a.NV, nvec = a.B * a.G;
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  const bool work = it < a.Hkv * a.nvt * 8 * NV;
  const int n = it % NV, c = (it / NV) & 7, ty = it / (NV * 8), y = ty % a.nvt, h = ty / a.nvt;
  const int vn = y * NV + n;
  uint4 u1 = make_uint4(0, 0, 0, 0), u2 = u1;
  if (work && vn < nvec) {
    const uint16_t* qp = a.q + (size_t)((vn / a.G) * a.Hq + h * a.G + vn % a.G) * kD + c * 8;
    u1 = ld_nc_u4(qp);
    u2 = ld_nc_u4(qp + kHalf);
  }
  __syncthreads();
  const uint32_t w1[4] = {u1.x, u1.y, u1.z, u1.w}, w2[4] = {u2.x, u2.y, u2.z, u2.w};
  uint16_t h1[8], l1[8], h2[8], l2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {  // half-split pair (m, m+64); zero rows stay zero
    const float x1 = (e & 1) ? bf_hi(w1[e >> 1]) : bf_lo(w1[e >> 1]);
    const float x2 = (e & 1) ? bf_hi(w2[e >> 1]) : bf_lo(w2[e >> 1]);
    const float2 cs = sbcs[c * 8 + e];
    umma::split_bf16(fmaf(x1, cs.x, -x2 * cs.y), h1[e], l1[e]);
    umma::split_bf16(fmaf(x2, cs.x, x1 * cs.y), h2[e], l2[e]);
  }
  pdl_wait();  // the previous step's LUT reads qt (and its attention the window table)
  pdl_trigger();
#ifdef A2ATS_PHASES
  if (threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_prep_tl[4096 + blockIdx.x][2] = t_;
  }
#endif
  if (!a.cs_in_lut)  // (else the persistent LUT's idle epilogue warps write it, off this kernel's path)
    for (int k = it; k < a.window * kHalf; k += gridDim.x * blockDim.x) {  // window table cs[r][m]
      double sn, cn;
      sincos((double)(k >> 6) * a.rt.inv_freq[k & (kHalf - 1)], &sn, &cn);
      a.cs[k] = make_float2((float)cn, (float)sn);
    }
  if (work) {
    uint4* dst = reinterpret_cast<uint4*>(a.qt + (size_t)ty * 32 * NV * 8);
    dst[c * NV + n] = pack8(h1);
    dst[(c + 8) * NV + n] = pack8(h2);
    dst[(c + 16) * NV + n] = pack8(l1);
    dst[(c + 24) * NV + n] = pack8(l2);
  }
#ifdef A2ATS_PHASES
  if (threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_prep_tl[4096 + blockIdx.x][1] = t_;
  }
#endif
}

// a2 on the FP32 pipes: LUT[b, hq, l] = q~ . c_l (Eq. 21) with q~ = q R_b (Eq. 12) in fp32,
// folded over the G query heads (Q10) into agg.  CTA = (128-codeword tile, KV head, tile of
// 32 query vectors); thread = codeword row (its 256-B codeword streamed in 16-element
// pieces); q~ rows in shared memory, read as broadcasts.  For contractions too small for the
// tensor cores to pay off (B*G*L up to ~1e5).  CTAs of vector tile 0 / head 0
// also write the window table cs[r][m] (fp64 angles), as the tensor LUT's CTAs do.
template <int G, int FV>
__global__ __launch_bounds__(128) void lut_fma_kernel(LutArgs a) {
  __shared__ __align__(16) float sq[FV][kD];
  __shared__ float2 sbcs[kHalf];
  const int tid = threadIdx.x, h = blockIdx.y, y = blockIdx.z;
  const int nvec = a.B * G, v0 = y * FV;
  const int l = blockIdx.x * 128 + tid;
  // the thread's codeword row (256 B), all loads in flight before the q~ build
  uint4 u[16];
  const uint16_t* cr = a.codebook + ((size_t)h * a.L + min(l, a.L - 1)) * kD;
#pragma unroll
  for (int i = 0; i < 16; ++i) u[i] = ld_nc_u4(cr + 8 * i);
  if (tid < kHalf) sbcs[tid] = a.bcs[tid];
  __syncthreads();
  {  // q~ rows of this tile (zero past B*G); all q loads in flight before use
    constexpr int kJ = FV * kHalf / 128;
    uint16_t x1[kJ], x2[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int it = tid + 128 * j, v = it >> 6, m = it & (kHalf - 1), vn = v0 + v;
      x1[j] = x2[j] = 0;
      if (vn < nvec) {
        const uint16_t* qp = a.q + (size_t)((vn / G) * a.Hq + h * G + vn % G) * kD;
        x1[j] = __ldg(qp + m);
        x2[j] = __ldg(qp + m + kHalf);
      }
    }
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int it = tid + 128 * j, v = it >> 6, m = it & (kHalf - 1);
      const float2 cs = sbcs[m];
      const float f1 = bf_u16(x1[j]), f2 = bf_u16(x2[j]);
      sq[v][m] = fmaf(f1, cs.x, -f2 * cs.y);
      sq[v][m + kHalf] = fmaf(f2, cs.x, f1 * cs.y);
    }
  }
  pdl_wait();  // the previous step's select reads agg, its attention the window table
  pdl_trigger();
  if (y == 0 && h == 0)
    for (int k = blockIdx.x * 128 + tid; k < a.window * kHalf; k += gridDim.x * 128) {
      double sn, cn;
      sincos((double)(k >> 6) * a.rt.inv_freq[k & (kHalf - 1)], &sn, &cn);
      a.cs[k] = make_float2((float)cn, (float)sn);
    }
  __syncthreads();
  if (l >= a.L) return;
  float acc[FV];
#pragma unroll
  for (int v = 0; v < FV; ++v) acc[v] = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float cf[8] = {bf_lo(u[i].x), bf_hi(u[i].x), bf_lo(u[i].y), bf_hi(u[i].y),
                         bf_lo(u[i].z), bf_hi(u[i].z), bf_lo(u[i].w), bf_hi(u[i].w)};
#pragma unroll
    for (int v = 0; v < FV; ++v) {
      const float4 qa = *reinterpret_cast<const float4*>(&sq[v][8 * i]);
      const float4 qb = *reinterpret_cast<const float4*>(&sq[v][8 * i + 4]);
      float t = acc[v];
      t = fmaf(cf[0], qa.x, t);
      t = fmaf(cf[1], qa.y, t);
      t = fmaf(cf[2], qa.z, t);
      t = fmaf(cf[3], qa.w, t);
      t = fmaf(cf[4], qb.x, t);
      t = fmaf(cf[5], qb.y, t);
      t = fmaf(cf[6], qb.z, t);
      t = fmaf(cf[7], qb.w, t);
      acc[v] = t;
    }
  }
  const bool sum = (a.group_reduce == A2ATS_GROUP_SUM);
#pragma unroll
  for (int v = 0; v < FV; ++v) {
    const int vn = v0 + v;
    if (vn < nvec && a.lut_full) a.lut_full[((size_t)(vn / G) * a.Hq + h * G + vn % G) * a.L + l] = acc[v];
  }
#pragma unroll
  for (int v = 0; v < FV; v += G) {  // fold groups of G consecutive vectors (G | FV)
    const int vn = v0 + v;
    if (vn < nvec) {
      float x = acc[v];
#pragma unroll
      for (int g = 1; g < G; ++g) x = sum ? x + acc[v + g] : fmaxf(x, acc[v + g]);
      a.agg[((size_t)(vn / G) * a.Hkv + h) * a.L + l] = x;
    }
  }
}

template <int G>
__global__ __launch_bounds__(128, 1) void prep_kernel(const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmC, PrepArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  A2ATS_TL(g_prep_tl, 0);
  int i = blockIdx.x;
  if (i < p.n_lut) {
    A2ATS_TL_VAL(g_prep_tl, 1);
    lut_tile<G>(tmA, p, i, smem);
  } else if ((i -= p.n_lut) < p.n_enc) {
    A2ATS_TL_VAL(g_prep_tl, 2);
    const int cx_n = (p.enc_tx + p.enc_tpc - 1) / p.enc_tpc, cx = i % cx_n;
    encode_tiles(tmC, p.enc, cx * p.enc_tpc, min(p.enc_tx, (cx + 1) * p.enc_tpc), i / cx_n, cx_n, p.enc_nv,
                 p.enc_cols, smem);
  } else {
    i -= p.n_enc;
    A2ATS_TL_VAL(g_prep_tl, 3);
    const int npairs = p.lut.B * p.lut.Hkv;
    const int pair0 = i * p.win_ppc;
    window_tile(p, pair0, max(0, min(p.win_ppc, npairs - pair0)), smem);
  }
  A2ATS_TL(g_prep_tl, 1);
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

template <int G>
cudaError_t launch_prep_g(const PrepArgs& p, const CUtensorMap& tmA, const CUtensorMap& tmC, cudaStream_t st) {
  const int smem = prep_smem_bytes(p);
  cudaError_t e = ensure_smem(prep_kernel<G>, smem);
  if (e != cudaSuccess) return e;
  const int n = p.n_lut + p.n_enc + p.n_win;
  if (n == 0) return cudaSuccess;
  return launch_pdl(prep_kernel<G>, dim3(n), dim3(128), smem, st, tmA, tmC, p);
}
}  // namespace

int prep_smem_bytes(const PrepArgs& p) {
  int smem = 0;
  if (p.n_lut) smem = max(smem, lut_tile_smem(p.lut.NV));
  if (p.n_enc) smem = max(smem, encode_tile_smem(p.enc_nv));
  if (p.n_win) smem = max(smem, kWinSmem);
  return smem + 1024;  // alignment slack for the SW128 slabs
}

template <int FV>
cudaError_t launch_lut_fma_fv(const LutArgs& la, cudaStream_t st) {
  const dim3 grid((la.L + 127) / 128, la.Hkv, (la.B * la.G + FV - 1) / FV);
  switch (la.G) {
    case 1: return launch_pdl(lut_fma_kernel<1, FV>, grid, dim3(128), 0, st, la);
    case 2: return launch_pdl(lut_fma_kernel<2, FV>, grid, dim3(128), 0, st, la);
    case 4: return launch_pdl(lut_fma_kernel<4, FV>, grid, dim3(128), 0, st, la);
    default: return launch_pdl(lut_fma_kernel<8, FV>, grid, dim3(128), 0, st, la);
  }
}
// vector tile of 8 for tiny batches, 16 otherwise (measured: a 32-vector tile runs at half
// the speed of two 16-vector tiles)
cudaError_t launch_lut_fma(const LutArgs& la, cudaStream_t st) {
  return la.B * la.G <= 8 ? launch_lut_fma_fv<8>(la, st) : launch_lut_fma_fv<16>(la, st);
}

template <int G>
cudaError_t launch_lut_persist_g(const LutArgs& la, const CUtensorMap& tmA, cudaStream_t st) {
  const int smem = lut_persist_smem(la.NV);
  cudaError_t e = ensure_smem(lut_persist_kernel<G>, smem);
  if (e != cudaSuccess) return e;
  const int ntx = (la.L + kTC - 1) / kTC, n_units = la.Hkv * la.nvt * ntx;
  const int grid = std::min(sm_count(), n_units);
  return launch_pdl(lut_persist_kernel<G>, dim3(grid), dim3(kLpWarps * 32), smem, st, tmA, la, n_units, ntx);
}
cudaError_t launch_lut_persist(const LutArgs& la, const CUtensorMap& tmA, cudaStream_t st) {
  switch (la.G) {
    case 1: return launch_lut_persist_g<1>(la, tmA, st);
    case 2: return launch_lut_persist_g<2>(la, tmA, st);
    case 4: return launch_lut_persist_g<4>(la, tmA, st);
    default: return launch_lut_persist_g<8>(la, tmA, st);
  }
}

size_t qprep_bytes(int Hkv, int nvt, int NV) { return (size_t)Hkv * nvt * 32 * NV * 16; }
cudaError_t launch_qprep(const LutArgs& la, cudaStream_t st) {
  const int n = la.Hkv * la.nvt * 8 * la.NV;
  return launch_pdl(qprep_kernel, dim3((n + 255) / 256), dim3(256), 0, st, la);
}

#ifndef A2ATS_LUT_NV_MAX
#define A2ATS_LUT_NV_MAX 128  // tuning define: widest query tile (MMA N) of the LUT
#endif
int lut_tile_nv(int nvec) { return nvec >= A2ATS_LUT_NV_MAX ? A2ATS_LUT_NV_MAX : ((nvec + 15) / 16) * 16; }  // MMA N: multiple of 16, <= 128 (B tile <= 64 KB)
int prep_lut_cols(int NV) { return (int)umma::tmem_cols_for(NV); }

cudaError_t launch_prep(const PrepArgs& p, const CUtensorMap& tmA, const CUtensorMap& tmC, cudaStream_t st) {
  switch (p.n_lut ? p.lut.G : 1) {
    case 1: return launch_prep_g<1>(p, tmA, tmC, st);
    case 2: return launch_prep_g<2>(p, tmA, tmC, st);
    case 4: return launch_prep_g<4>(p, tmA, tmC, st);
    default: return launch_prep_g<8>(p, tmA, tmC, st);
  }
}

cudaError_t launch_scores(const float* lut_full, const uint16_t* codes, float* scores, int B, int Hq, int Hkv,
                          int G, int L, int n_max, int n_ctx, cudaStream_t st) {
  dim3 grid((n_ctx + 1023) / 1024, B * Hq);
  return launch_pdl(scores_kernel, grid, dim3(256), 0, st, lut_full, codes, scores, Hq, Hkv, G, L, n_max, n_ctx);
}

}  // namespace a2ats

A2ATS_PHASE_EXPORT(a2ats_debug_lut_phases, a2ats::g_lut_phase)
A2ATS_TL_EXPORT(a2ats_debug_prep_timeline, a2ats::g_prep_tl)
