// a0: query-aware VQ encoding of keys (Eq. 14; Eq. 20).
//
//   f'(k; C) = argmin_j (k - c_j) H (k - c_j)^T = argmin_j ( n_j - 2 k . c^_j )
// with S = (H + H^T) / 2, c^_j = c_j S and n_j = c_j H c_j^T (k H k^T does not
// depend on j).  prepare_kernel computes n_j and c^_j once per codebook (offline
// state, a2ats_qavq_prepare); c^_j is stored as a bf16 hi + lo pair so that one
// tensor-core pass over K = 2 x 128 reproduces k . c^_j to ~2^-16 relative (keys
// are exact in bf16).  No per-step key transform is needed.
//
//   decode-time encode tile (encode_common.cuh, run as a role of prep_kernel; few
//     keys per head): codewords on the MMA M side, 128 per CTA, all keys of the
//     head on N; argmin epilogue reduces the rows (codewords) of each key column
//     across lanes and warps, CTAs of a head combine by 64-bit atomicMax on the
//     complemented (ordered dist, index) word; the last CTA of the head writes
//     codes and histogram.
//   encode_bulk_kernel (prefill): 128 keys on M, 128-codeword tiles on N streamed
//     through a double buffer, per-key running argmin in registers; CTAs that split
//     the codebook combine the same way.
// Ties resolve to the lowest codeword index (reading Q12): the in-thread scan visits
// codewords in increasing order with a strict '<', lane / warp reductions pick the
// lowest index among equal distances, and the 64-bit combine orders by (dist, index),
// so the result is deterministic.
#include "encode_common.cuh"

namespace a2ats {

namespace {
constexpr int kTV = 128;   // keys per CTA in the bulk kernel (MMA M)
constexpr int kBulkSmem = 1024 + kTV * kD * 2 + 2 * kCW * kRowB + 2 * kCW * 4;  // align + A + 2 x B + 2 x n_j


// c^_j = c_j S, n_j = c^_j . c_j (= c_j H c_j^T); one warp per codeword, S in smem.
__global__ __launch_bounds__(256) void prepare_kernel(const uint16_t* __restrict__ codebook, const float* __restrict__ H,
                                                      float* __restrict__ nrm, uint16_t* __restrict__ chat, int L) {
  extern __shared__ __align__(16) float Ss[];  // [128][128] symmetrised H, or unused
  __shared__ float crow[8][kD];
  const int h = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (H) {
    const float* Hh = H + (size_t)h * kD * kD;
    for (int i = tid; i < kD * kD; i += 256) {
      const int d = i >> 7, e = i & (kD - 1);
      Ss[i] = 0.5f * (Hh[d * kD + e] + Hh[e * kD + d]);
    }
  }
  __syncthreads();
  for (int c = blockIdx.x * 64 + warp; c < min(L, blockIdx.x * 64 + 64); c += 8) {
    const uint16_t* cp = codebook + ((size_t)h * L + c) * kD;
#pragma unroll
    for (int i = 0; i < 4; ++i) crow[warp][lane + 32 * i] = bf_u16(cp[lane + 32 * i]);
    __syncwarp();
    float part = 0.f;
    uint16_t* dst = chat + ((size_t)h * L + c) * (2 * kD);
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int e = lane + 32 * k;
      float ce = crow[warp][e];
      if (H) {
        ce = 0.f;
        for (int d = 0; d < kD; ++d) ce = fmaf(crow[warp][d], Ss[d * kD + e], ce);
      }
      part = fmaf(ce, crow[warp][e], part);
      uint16_t hi, lo;
      umma::split_bf16(ce, hi, lo);
      dst[e] = hi;
      dst[kD + e] = lo;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if (lane == 0) nrm[(size_t)h * L + c] = part;
    __syncwarp();
  }
}


// grid (ceil(nvec / 128), Hkv, splits); CTA = 128 keys x codeword tiles [tbeg, tend) of 128.
__global__ __launch_bounds__(128, 1) void encode_bulk_kernel(const __grid_constant__ CUtensorMap tmC, EncArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB0 = smem;                         // 2 x 4 SW128 K slabs [128 codewords][128 B]
  uint8_t* sA = smem + 2 * kCW * kRowB;        // [16 chunks][128 keys][16 B]
  float* sN0 = reinterpret_cast<float*>(sA + kTV * kD * 2);  // 2 x [128] n_j
  __shared__ uint64_t mbar, tbar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int h = blockIdx.y, split = blockIdx.z;
  const int vec0 = blockIdx.x * kTV;
  const int ntile = (a.L + kCW - 1) / kCW;
  const int tbeg = split * a.tiles_per_split, tend = min(ntile, tbeg + a.tiles_per_split);

  if (warp == 0) umma::tmem_alloc<kCW>(&tslot);
  if (tid == 0) {
    umma::mbar_init(&mbar, 1);
    umma::mbar_init(&tbar[0], 1);
    umma::mbar_init(&tbar[1], 1);
    umma::mbar_fence_init();
    issue_chat_tile(tmC, a, h, tbeg * kCW, sB0, &tbar[0]);
  }
  for (int idx = tid; idx < kTV * 16; idx += 128) {  // keys: exact bf16, canonical K-major
    const int r = idx >> 4, c = idx & 15;
    uint8_t* d = sA + (c * kTV + r) * 16;
    if (vec0 + r < a.nvec) cp_async16(d, key_row(a, h, vec0 + r) + c * 8);
    else *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
  }
  load_nrm(a, h, tbeg * kCW, sN0);
  cp_async_commit();
  pdl_wait();
  pdl_trigger();

  float best = INFINITY;
  int bidx = 0x7fffffff;
  const uint32_t idesc = umma::idesc_bf16(kTV, kCW);
#pragma unroll 1
  for (int tile = tbeg; tile < tend; ++tile) {
    const int buf = (tile - tbeg) & 1;
    if (tile + 1 < tend) {  // the other buffer was released by the previous iteration's barrier
      if (tid == 0) issue_chat_tile(tmC, a, h, (tile + 1) * kCW, sB0 + (buf ^ 1) * (kCW * kRowB), &tbar[buf ^ 1]);
      load_nrm(a, h, (tile + 1) * kCW, sN0 + (buf ^ 1) * kCW);
    }
    cp_async_wait<0>();  // keys (first iteration)
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
      umma::mbar_wait(&tbar[buf], ((tile - tbeg) >> 1) & 1);
      const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB0 + buf * (kCW * kRowB));
#pragma unroll
      for (int s = 0; s < 16; ++s) {  // keys against c^_hi (slabs 0, 1), then against c^_lo (2, 3)
        const uint64_t ad = umma::sdesc(aBase + (2 * (s & 7)) * (kTV * 16), kTV * 16, 128);
        const uint64_t bd = chat_desc(bBase, s);
        umma::mma_bf16(tmem, ad, bd, idesc, s > 0 ? 1u : 0u);
      }
      umma::commit(&mbar);
    }
    __syncwarp();
    umma::mbar_wait(&mbar, (tile - tbeg) & 1);
    umma::fence_after();
    const float* sN = sN0 + buf * kCW;
    const int c0 = tile * kCW;
#pragma unroll 1
    for (int col0 = 0; col0 < kCW; col0 += 32) {
      uint32_t r[2][16];
      umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + col0, r[0]);
      umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + col0 + 16, r[1]);
      umma::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int code = c0 + col0 + i;
        const float dist = fmaf(-2.f, __uint_as_float(r[i >> 4][i & 15]), sN[col0 + i]);
        if (code < a.L && dist < best) {  // codewords visited in increasing order
          best = dist;
          bidx = code;
        }
      }
    }
    umma::fence_before();
    __syncthreads();  // TMEM and this B buffer are free again
  }
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<kCW>(tslot);
  const int nv = min(kTV, a.nvec - vec0);
  combine_and_finalize(a, h, vec0, nv, a.counter + (size_t)h * gridDim.x + blockIdx.x, gridDim.z, tid < nv,
                       pack_dist(ordered_key(best), bidx));
}

}  // namespace

cudaError_t launch_prepare(const uint16_t* codebook, const float* H, float* nrm, uint16_t* chat, int Hkv, int L,
                           cudaStream_t st) {
  const int smem = H ? kD * kD * 4 : 0;
  cudaError_t e = cudaFuncSetAttribute(prepare_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kD * kD * 4);
  if (e != cudaSuccess) return e;
  dim3 grid((L + 63) / 64, Hkv);
  prepare_kernel<<<grid, 256, smem, st>>>(codebook, H, nrm, chat, L);
  return cudaGetLastError();
}

// Prefill encoder (more than encode_cw_max() keys per head); fewer keys go through the
// decode-time encode role of the step kernel (prep.cu).
cudaError_t launch_encode_bulk(const EncArgs& a, const CUtensorMap& tm, cudaStream_t st) {
  cudaError_t e = ensure_smem(encode_bulk_kernel, kBulkSmem);
  if (e != cudaSuccess) return e;
  const int ntile = (a.L + kCW - 1) / kCW;
  dim3 grid((a.nvec + kTV - 1) / kTV, a.Hkv, (ntile + a.tiles_per_split - 1) / a.tiles_per_split);
  return launch_pdl(encode_bulk_kernel, grid, dim3(128), kBulkSmem, st, tm, a);
}

int encode_codeword_tile() { return kCW; }
int encode_key_tile() { return kTV; }
int encode_cw_max() { return 256; }

}  // namespace a2ats

