// Shared pieces of the QAVQ encoders (a0; Eq. 14, Eq. 20):
// included by encode.cu (prefill encoder) and prep.cu (the decode-time encode role of
// the step's first kernel).  See encode.cu for the formulation.
#pragma once
#include "internal.cuh"
#include "umma.cuh"

namespace a2ats {
namespace {
constexpr int kCW = 128;           // codewords per tile (MMA M in the decode tile, MMA N in the bulk kernel)
constexpr int kRowB = 2 * kD * 2;  // bytes of one prepared codeword row (hi | lo bf16)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ unsigned long long pack_dist(uint32_t okey, int code) {
  return ((unsigned long long)okey << 32) | (unsigned)code;
}

__device__ __forceinline__ void finalize_code(const EncArgs& a, int h, int v, unsigned long long packed) {
  const int code = (int)(packed & 0xffffffffull);
  const int b = v / a.T, t = a.t_begin + (v - b * a.T);
  const size_t pair = (size_t)b * a.Hkv + h;
  if (a.codes8) a.codes8[pair * a.n_max + t] = (uint8_t)code;
  else a.codes[pair * a.n_max + t] = (uint16_t)code;
  if (a.hist) atomicAdd(a.hist + pair * a.L + code, 1);
}

// Global row of key vector v of head h: v = b * T + (t - t_begin).
__device__ __forceinline__ const uint16_t* key_row(const EncArgs& a, int h, int v) {
  const int b = v / a.T, t = a.t_begin + (v - b * a.T);
  return a.keys + (((size_t)b * a.Hkv + h) * a.n_max + t) * kD;
}

// Prepared codeword tile: rows h*L + c0 .. (+128) of chat, 4 TMA boxes of 64 columns
// (c^_hi 0..63, c^_hi 64..127, c^_lo 0..63, c^_lo 64..127) into four SW128 K slabs of
// 16 KB; one thread issues, completion on tbar.  Rows past the head belong to the
// next head (or are zero-filled) and are never selected (code < L checks).
__device__ __forceinline__ void issue_chat_tile(const CUtensorMap& tm, const EncArgs& a, int h, int c0, uint8_t* dst,
                                                uint64_t* tbar) {
  umma::mbar_expect_tx(tbar, kCW * kRowB);
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) umma::tma_load_2d(dst + k4 * (kCW * 128), &tm, 64 * k4, h * a.L + c0, tbar);
}
__device__ __forceinline__ void load_nrm(const EncArgs& a, int h, int c0, float* sN) {
  for (int i = threadIdx.x; i < kCW; i += blockDim.x) sN[i] = (c0 + i < a.L) ? __ldg(a.nrm + (size_t)h * a.L + c0 + i) : 0.f;
}
// MMA k-step s (16 elements) of a chat tile: slab s / 4, 32 B per step inside the slab
__device__ __forceinline__ uint64_t chat_desc(uint32_t base, int s) {
  return umma::sdesc_sw128(base + (s >> 2) * (kCW * 128) + (s & 3) * 32);
}

// Cross-CTA combine of (ordered dist, code) per key, then the last CTA of the
// group [counter] finalises codes / histogram and resets its slots.
__device__ void combine_and_finalize(const EncArgs& a, int h, int v0, int nv, unsigned int* counter, int nparts,
                                     bool have, unsigned long long mine) {
  const int tid = threadIdx.x;
  if (nparts == 1) {
    if (have) finalize_code(a, h, v0 + tid, mine);
    return;
  }
  if (have) atomicMax(a.slot + (size_t)h * a.nvec + v0 + tid, ~mine);
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(counter, 1u) == (unsigned)nparts - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int i = tid; i < nv; i += blockDim.x) {
    unsigned long long* sp = a.slot + (size_t)h * a.nvec + v0 + i;
    finalize_code(a, h, v0 + i, ~__ldcg(sp));
    *sp = 0ull;
  }
  if (tid == 0) *counter = 0u;
}

// Decode-time encode (few keys per head): code tiles [xt0, xt1) (128 codewords each) of KV
// head h, one after the other through one TMA buffer, on the MMA M side; the head's nvec
// (<= 256) keys on N (NV = nvec rounded up to 16, ncols = TMEM columns, a power of two
// >= max(32, NV)).  nparts = CTAs of the head (they combine through the slots).  smem:
// 1024-aligned, encode_tile_smem(NV) bytes.
__host__ __device__ constexpr int encode_tile_smem(int NV) { return kCW * kRowB + NV * kD * 2 + kCW * 4 + 4 * NV * 8; }
__device__ __forceinline__ void encode_tiles(const CUtensorMap& tmC, const EncArgs& a, int xt0, int xt1, int h,
                                             int nparts, int NV, uint32_t ncols, uint8_t* smem) {
  uint8_t* sA = smem;                           // 4 SW128 K slabs [128 codewords][128 B]
  uint8_t* sB = smem + kCW * kRowB;             // [16 chunks][NV keys][16 B]
  float* sN = reinterpret_cast<float*>(sB + NV * kD * 2);                    // [128] n_j
  unsigned long long* red = reinterpret_cast<unsigned long long*>(sN + kCW);  // [4][NV] per-warp best
  __shared__ uint64_t mbar, tbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) umma::tmem_alloc_n(&tslot, ncols);
  if (tid == 0) {
    umma::mbar_init(&mbar, 1);
    umma::mbar_init(&tbar, 1);
    umma::mbar_fence_init();
    issue_chat_tile(tmC, a, h, xt0 * kCW, sA, &tbar);  // prepared codewords (offline state)
  }
  // this step's keys (written before the call)
  for (int idx = tid; idx < NV * 16; idx += 128) {
    const int n = idx >> 4, c = idx & 15;
    uint8_t* d = sB + (c * NV + n) * 16;
    if (n < a.nvec) cp_async16(d, key_row(a, h, n) + c * 8);
    else *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
  }
  cp_async_commit();
  for (int i = tid; i < 4 * NV; i += 128) red[i] = ~0ull;
  cp_async_wait<0>();
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = umma::idesc_bf16(kCW, NV);
#pragma unroll 1
  for (int xt = xt0; xt < xt1; ++xt) {
    const int it = xt - xt0, code0 = xt * kCW;
    load_nrm(a, h, code0, sN);
    if (tid == 0) {
      umma::mbar_wait(&tbar, it & 1);
      const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
#pragma unroll
      for (int s = 0; s < 16; ++s) {  // K = 256: c^_hi (slabs 0, 1) then c^_lo (slabs 2, 3), same keys
        const uint64_t ad = chat_desc(aBase, s);
        const uint64_t bd = umma::sdesc(bBase + (2 * (s & 7)) * (NV * 16), NV * 16, 128);
        umma::mma_bf16(tmem, ad, bd, idesc, s > 0 ? 1u : 0u);
      }
      umma::commit(&mbar);
    }
    __syncwarp();
    umma::mbar_wait(&mbar, it & 1);
    umma::fence_after();
    if (tid == 0 && xt + 1 < xt1) issue_chat_tile(tmC, a, h, code0 + kCW, sA, &tbar);  // sA is free again
    __syncthreads();  // n_j of this tile
    // epilogue: thread <-> codeword row; per key column, argmin over the rows (running best per warp)
    const int row = warp * 32 + lane;
    const bool valid = code0 + row < a.L;
    const float nj = sN[row];
#pragma unroll 1
    for (int col0 = 0; col0 < NV; col0 += 16) {
      uint32_t r[16];
      umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + col0, r);
      umma::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t key = valid ? ordered_key(fmaf(-2.f, __uint_as_float(r[i]), nj)) : 0xffffffffu;
        const uint32_t wmin = __reduce_min_sync(0xffffffffu, key);
        const uint32_t hit = __ballot_sync(0xffffffffu, key == wmin);  // lowest lane = lowest codeword
        if (lane == 0) {
          unsigned long long* rp = red + warp * NV + col0 + i;
          *rp = min(*rp, pack_dist(wmin, code0 + warp * 32 + __ffs(hit) - 1));
        }
      }
    }
    umma::fence_before();
    __syncthreads();  // TMEM read out and sN consumed before the next tile
    umma::fence_after();
  }
  if (warp == 0) umma::tmem_dealloc_n(tmem, ncols);
  pdl_wait();  // slots / codes / hist are written below (the MMA work above only read step inputs)
  pdl_trigger();  // after the wait, like every kernel of the path (internal.cuh invariant)
  // tid <-> key column (nvec <= 256: two passes at most)
  for (int base = 0; base < a.nvec; base += 128) {
    const int v = base + tid;
    unsigned long long best = ~0ull;
    if (v < a.nvec) {
#pragma unroll
      for (int w = 0; w < 4; ++w) best = min(best, red[w * NV + v]);
    }
    combine_and_finalize(a, h, base, min(128, a.nvec - base), a.counter + h * 2 + (base >> 7), nparts,
                         v < a.nvec, best);
  }
}

}  // namespace
}  // namespace a2ats
