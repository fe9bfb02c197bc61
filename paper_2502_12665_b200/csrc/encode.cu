// a0: query-aware VQ encoding of keys (Eq. 14; Eq. 20).
//
//   f'(k; C) = argmin_j (k - c_j) H (k - c_j)^T = argmin_j ( n_j - 2 (k H) . c_j )
// with n_j = c_j H c_j^T (a2ats_qavq_prepare) because H is symmetric.
//   keyh_kernel   : u = k H (d x d per key, CUDA cores, fp32)
//   encode_kernel : u . c_j for 128 keys x 256 codewords per tcgen05 tile
//                   (A = u split hi/lo in bf16, B = bf16 codebook tile, fp32
//                   accumulator in TMEM), argmin epilogue per key row.
// Ties resolve to the lowest codeword index (reading Q12): the per-thread scan
// visits codewords in increasing order with a strict '<', and partial results of
// CTAs that split the codebook are combined by 64-bit atomicMax on the
// complemented (ordered dist, index) word, which is order independent, so the
// result is deterministic.
#include "internal.cuh"
#include "umma.cuh"

namespace a2ats {

namespace {
constexpr int kTV = 128;   // keys per CTA (MMA M)
constexpr int kNB = 256;   // codewords per MMA tile (MMA N)
constexpr int kEncSmem = kTV * 2 * kD * 2 + 2 * kNB * kD * 2 + 2 * kNB * 4;  // A + 2 x B + 2 x nrm

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

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

// u[h][v][e] = sum_d k[b][h][t][d] H[h][d][e]  (v = b*T + t - t_begin); u = k when H == nullptr.
// 16 keys x 128 outputs per CTA of 256 threads; H[h] staged in shared memory with all
// 128-bit loads in flight at once (the kernel is latency-bound at decode sizes).
constexpr int kKeyhV = 16;
__global__ __launch_bounds__(256) void keyh_kernel(EncArgs a) {
  extern __shared__ __align__(16) float Hs[];  // [128][128]
  __shared__ float ks[kKeyhV][kD];
  const int h = blockIdx.y, tid = threadIdx.x;
  const int v0 = blockIdx.x * kKeyhV;
  if (a.H) {
    const float4* src = reinterpret_cast<const float4*>(a.H + (size_t)h * kD * kD);
    float4 tmp[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) tmp[i] = __ldg(src + tid + 256 * i);
#pragma unroll
    for (int i = 0; i < 16; ++i) reinterpret_cast<float4*>(Hs)[tid + 256 * i] = tmp[i];
  }
  for (int i = tid; i < kKeyhV * 16; i += 256) {  // 16 keys x 16 chunks of 8 bf16
    const int vv = i >> 4, c = i & 15;
    const int v = v0 + vv;
    uint4 x = make_uint4(0, 0, 0, 0);
    if (v < a.nvec) {
      const int b = v / a.T, t = a.t_begin + (v - b * a.T);
      x = ld_nc_u4(a.keys + (((size_t)b * a.Hkv + h) * a.n_max + t) * kD + c * 8);
    }
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) ks[vv][c * 8 + j] = (j & 1) ? bf_hi(w[j >> 1]) : bf_lo(w[j >> 1]);
  }
  __syncthreads();
  pdl_wait();  // H and the keys are step inputs; u is read by the previous step's encode
  pdl_trigger();
  const int e = tid & (kD - 1), vh = tid >> 7;  // 2 groups of 8 keys
  float acc[8];
  if (a.H) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll 8
    for (int d = 0; d < kD; ++d) {
      const float hd = Hs[d * kD + e];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(ks[vh * 8 + i][d], hd, acc[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = ks[vh * 8 + i][e];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int v = v0 + vh * 8 + i;
    if (v < a.nvec) a.u[((size_t)h * a.nvec + v) * kD + e] = acc[i];
  }
}

__device__ __forceinline__ unsigned long long pack_dist(float dist, int code) {
  return ((unsigned long long)ordered_key(dist) << 32) | (unsigned)code;
}

__device__ __forceinline__ void finalize_code(const EncArgs& a, int h, int v, unsigned long long packed) {
  const int code = (int)(packed & 0xffffffffull);
  const int b = v / a.T, t = a.t_begin + (v - b * a.T);
  const size_t pair = (size_t)b * a.Hkv + h;
  a.codes[pair * a.n_max + t] = (uint16_t)code;
  if (a.hist) atomicAdd(a.hist + pair * a.L + code, 1);
}

// grid (ceil(nvec/128), Hkv, splits); CTA = 128 keys x codeword tiles [tbeg, tend) of 256
__global__ __launch_bounds__(128, 1) void encode_kernel(EncArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                                  // [32 chunks][128 keys][16 B]: hi 0..15, lo 16..31
  uint8_t* sB0 = smem + kTV * 2 * kD * 2;              // 2 x [16 chunks][256 codes][16 B]
  float* sN0 = reinterpret_cast<float*>(sB0 + 2 * kNB * kD * 2);  // 2 x [256] codeword norms n_j
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y, split = blockIdx.z;
  const int vec0 = blockIdx.x * kTV;
  const int ntile = (a.L + kNB - 1) / kNB;
  const int tbeg = split * a.tiles_per_split, tend = min(ntile, tbeg + a.tiles_per_split);

  if (warp == 0) umma::tmem_alloc<256>(&tslot);
  if (tid == 0) {
    umma::mbar_init(&mbar, 1);
    umma::mbar_fence_init();
  }

  auto load_tile = [&](int tile, int buf) {
    uint8_t* sB = sB0 + buf * (kNB * kD * 2);
    const int c0 = tile * kNB;
    for (int idx = tid; idx < kNB * 16; idx += 128) {
      const int r = idx >> 4, c = idx & 15;
      uint8_t* dst = sB + (c * kNB + r) * 16;
      if (c0 + r < a.L) cp_async16(dst, a.codebook + ((size_t)h * a.L + c0 + r) * kD + c * 8);
      else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
    if (c0 + kNB <= a.L && (a.L & 3) == 0) {
      if (tid < kNB / 4) cp_async16(sN0 + buf * kNB + 4 * tid, a.nrm + (size_t)h * a.L + c0 + 4 * tid);
    } else {
      for (int i = tid; i < kNB; i += 128) sN0[buf * kNB + i] = (c0 + i < a.L) ? a.nrm[(size_t)h * a.L + c0 + i] : 0.f;
    }
    cp_async_commit();
  };
  load_tile(tbeg, 0);  // codebook tile + n_j: inputs, overlaps keyh's tail
  pdl_wait();          // u comes from keyh
  pdl_trigger();

  // A: key rows u (fp32) staged through the (still idle) second B buffer with cp.async,
  // then split into hi/lo bf16 chunks; this thread converts its own row.
  {
    uint8_t* stage = sB0 + kNB * kD * 2;  // 64 KB = 128 rows x 512 B
    const int nrow = min(kTV, a.nvec - vec0);
    for (int p = tid; p < nrow * 32; p += 128) {
      const int r = p >> 5, piece = p & 31;
      cp_async16(stage + r * 512 + piece * 16, a.u + ((size_t)h * a.nvec + vec0 + r) * kD + piece * 4);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const int v = vec0 + tid;
    const float4* up = reinterpret_cast<const float4*>(stage + tid * 512);
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
      float x[8];
      if (v < a.nvec) {
        const float4 p0 = up[2 * c], p1 = up[2 * c + 1];
        x[0] = p0.x; x[1] = p0.y; x[2] = p0.z; x[3] = p0.w; x[4] = p1.x; x[5] = p1.y; x[6] = p1.z; x[7] = p1.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = 0.f;
      }
      uint16_t hi[8], lo[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) umma::split_bf16(x[i], hi[i], lo[i]);
      *reinterpret_cast<uint4*>(sA + (c * kTV + tid) * 16) =
          make_uint4(hi[0] | (uint32_t(hi[1]) << 16), hi[2] | (uint32_t(hi[3]) << 16), hi[4] | (uint32_t(hi[5]) << 16),
                     hi[6] | (uint32_t(hi[7]) << 16));
      *reinterpret_cast<uint4*>(sA + ((16 + c) * kTV + tid) * 16) =
          make_uint4(lo[0] | (uint32_t(lo[1]) << 16), lo[2] | (uint32_t(lo[3]) << 16), lo[4] | (uint32_t(lo[5]) << 16),
                     lo[6] | (uint32_t(lo[7]) << 16));
    }
    __syncthreads();  // the staging buffer is refilled with codeword tiles below
  }

  float best = INFINITY;
  int bidx = 0x7fffffff;
  const uint32_t idesc = umma::idesc_bf16(kTV, kNB);
  for (int tile = tbeg; tile < tend; ++tile) {
    const int buf = (tile - tbeg) & 1;
    if (tile + 1 < tend) {
      load_tile(tile + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
      const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB0 + buf * (kNB * kD * 2));
#pragma unroll
      for (int s = 0; s < 16; ++s) {  // K = 256: u_hi against chunks 0..15, u_lo against the same B
        const uint64_t ad = umma::sdesc(aBase + (2 * s) * (kTV * 16), kTV * 16, 128);
        const uint64_t bd = umma::sdesc(bBase + (2 * (s & 7)) * (kNB * 16), kNB * 16, 128);
        umma::mma_bf16(tmem, ad, bd, idesc, s > 0 ? 1u : 0u);
      }
      umma::commit(&mbar);
    }
    __syncwarp();
    umma::mbar_wait(&mbar, (tile - tbeg) & 1);
    umma::fence_after();
    const float* sN = sN0 + buf * kNB;
    const int c0 = tile * kNB;
#pragma unroll 1
    for (int col0 = 0; col0 < kNB; col0 += 64) {  // 4 TMEM loads in flight, then one wait
      uint32_t r[4][16];
#pragma unroll
      for (int q = 0; q < 4; ++q) umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + col0 + 16 * q, r[q]);
      umma::tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int code = c0 + col0 + 16 * q + i;
          const float dist = fmaf(-2.f, __uint_as_float(r[q][i]), sN[col0 + 16 * q + i]);
          if (code < a.L && dist < best) {  // codewords visited in increasing order
            best = dist;
            bidx = code;
          }
        }
    }
    umma::fence_before();
    __syncthreads();  // TMEM and this B buffer are free again
  }

  const int v = vec0 + tid;
  const bool single = (gridDim.z == 1);
  if (v < a.nvec) {
    const unsigned long long pk = pack_dist(best, bidx);
    if (single) finalize_code(a, h, v, pk);
    else atomicMax(a.slot + (size_t)h * a.nvec + v, ~pk);
  }
  if (!single) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const unsigned prev = atomicAdd(a.counter + (size_t)h * gridDim.x + blockIdx.x, 1u);
      s_last = (prev == gridDim.z - 1);
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (v < a.nvec) {
        unsigned long long* sp = a.slot + (size_t)h * a.nvec + v;
        finalize_code(a, h, v, ~__ldcg(sp));
        *sp = 0ull;
      }
      if (tid == 0) a.counter[(size_t)h * gridDim.x + blockIdx.x] = 0u;
    }
  }
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<256>(tslot);
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
    cudaError_t e = cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kEncSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(keyh_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kD * kD * 4);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  dim3 g1((a.nvec + kKeyhV - 1) / kKeyhV, a.Hkv);
  cudaError_t e = launch_pdl(keyh_kernel, g1, dim3(256), a.H ? kD * kD * 4 : 0, st, a);
  if (e != cudaSuccess) return e;
  const int ntile = (a.L + kNB - 1) / kNB;
  dim3 g2((a.nvec + kTV - 1) / kTV, a.Hkv, (ntile + a.tiles_per_split - 1) / a.tiles_per_split);
  return launch_pdl(encode_kernel, g2, dim3(128), kEncSmem, st, a);
}

int encode_codeword_tile() { return kNB; }
int encode_key_tile() { return kTV; }

}  // namespace a2ats
