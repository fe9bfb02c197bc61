// Random-row gather bandwidth probe (tools only, not product code).
// Gathers `rows` random 256-B rows (x2: K and V) out of a large bf16 cache the
// way the attention kernel does, with three loaders, and reports GB/s:
//   ldg   : 128-bit loads into registers (8 in flight per lane)
//   cpas  : cp.async 16 B pieces into a per-warp smem ring (3 stages)
//   bulk  : cp.async.bulk (TMA 1D) of whole 256-B rows, mbarrier completion
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#include <cuda.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_ldg(const uint4* __restrict__ kc, const uint4* __restrict__ vc, const int* __restrict__ idx, int nrows, uint4* sink) {
  // each warp: 2 rows per step (16 lanes per row, 16 B each) for K and V
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r0 = gw * 16; r0 < nrows; r0 += nw * 16) {
    uint4 v[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + 2 * i + (lane >> 4);
      const int t = idx[min(r, nrows - 1)];
      v[2 * i] = kc[(size_t)t * 16 + (lane & 15)];
      v[2 * i + 1] = vc[(size_t)t * 16 + (lane & 15)];
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) { acc.x ^= v[i].x; acc.y ^= v[i].y; acc.z ^= v[i].z; acc.w ^= v[i].w; }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

__device__ __forceinline__ void cp16(void* s, const void* g) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(g) : "memory");
}

template <int ST, bool IL = false>
__global__ void k_cpas(const uint8_t* __restrict__ kc, const uint8_t* __restrict__ vc, const int* __restrict__ idx, int nrows, uint4* sink) {
  extern __shared__ uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = sm + warp * ST * 8192;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int ntiles = (nrows + 15) / 16;
  const int mytiles = (ntiles - gw + nw - 1) / nw;
  auto issue = [&](int s) {
    if (s < mytiles) {
      const int tile = gw + s * nw;
      uint8_t* st = ring + (s % ST) * 8192;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int p = lane + 32 * i;
        const int kv = p >> 8, row = (p >> 4) & 15, ch = p & 15;
        const int t = idx[min(tile * 16 + row, nrows - 1)];
        const uint8_t* src = IL ? kc + (size_t)t * 512 + kv * 256 + ch * 16 : (kv ? vc : kc) + (size_t)t * 256 + ch * 16;
        cp16(st + kv * 4096 + row * 256 + ch * 16, src);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < ST - 1; ++s) issue(s);
  uint32_t acc = 0;
  for (int s = 0; s < mytiles; ++s) {
    issue(s + ST - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 1) : "memory");
    __syncwarp();
    acc ^= *reinterpret_cast<const uint32_t*>(ring + (s % ST) * 8192 + lane * 16);
    __syncwarp();
  }
  if (acc == 0x12345678) sink[0] = make_uint4(acc, 0, 0, 0);
}

__device__ __forceinline__ void mbar_init(uint64_t* m, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* s, const void* g, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(m)) : "memory");
}

template <int ST>
__global__ void k_bulk(const uint8_t* __restrict__ kc, const uint8_t* __restrict__ vc, const int* __restrict__ idx, int nrows, uint4* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mb[8][ST];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = sm + warp * ST * 8192;
  if (lane == 0) for (int s = 0; s < ST; ++s) mbar_init(&mb[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int ntiles = (nrows + 15) / 16;
  const int mytiles = (ntiles - gw + nw - 1) / nw;
  auto issue = [&](int s) {
    if (s < mytiles) {
      const int tile = gw + s * nw;
      uint8_t* st = ring + (s % ST) * 8192;
      // 32 lanes: lane -> (kv, row); one 256-B bulk copy each
      const int kv = lane >> 4, row = lane & 15;
      const int t = idx[min(tile * 16 + row, nrows - 1)];
      if (lane == 0) mbar_expect(&mb[warp][s % ST], 8192);
      __syncwarp();
      bulk(st + kv * 4096 + row * 256, (kv ? vc : kc) + (size_t)t * 256, 256, &mb[warp][s % ST]);
    }
  };
  for (int s = 0; s < ST - 1; ++s) issue(s);
  uint32_t acc = 0;
  for (int s = 0; s < mytiles; ++s) {
    issue(s + ST - 1);
    mbar_wait(&mb[warp][s % ST], (s / ST) & 1);
    acc ^= *reinterpret_cast<const uint32_t*>(ring + (s % ST) * 8192 + lane * 16);
    __syncwarp();
  }
  if (acc == 0x12345678) sink[0] = make_uint4(acc, 0, 0, 0);
}


template <int ST>
__global__ void k_g4(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, const int* __restrict__ idx, int nrows, uint4* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mb[8][ST];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = sm + warp * ST * 8192;
  if (lane == 0) for (int s = 0; s < ST; ++s) mbar_init(&mb[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int ntiles = (nrows + 15) / 16;
  const int mytiles = (ntiles - gw + nw - 1) / nw;
  auto issue = [&](int s) {
    if (s < mytiles) {
      const int tile = gw + s * nw;
      uint8_t* st = ring + (s % ST) * 8192;
      const int t = idx[min(tile * 16 + (lane & 15), nrows - 1)];
      int rows[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) rows[i] = __shfl_sync(0xffffffffu, t, i);
      if (lane == 0) {
        mbar_expect(&mb[warp][s % ST], 8192);
        const uint32_t mbs = (uint32_t)__cvta_generic_to_shared(&mb[warp][s % ST]);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint32_t dk = (uint32_t)__cvta_generic_to_shared(st + g * 1024);
          const uint32_t dv = (uint32_t)__cvta_generic_to_shared(st + 4096 + g * 1024);
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                       :: "r"(dk), "l"(&tmk), "r"(0), "r"(rows[4*g]), "r"(rows[4*g+1]), "r"(rows[4*g+2]), "r"(rows[4*g+3]), "r"(mbs) : "memory");
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                       :: "r"(dv), "l"(&tmv), "r"(0), "r"(rows[4*g]), "r"(rows[4*g+1]), "r"(rows[4*g+2]), "r"(rows[4*g+3]), "r"(mbs) : "memory");
        }
      }
    }
  };
  for (int s = 0; s < ST - 1; ++s) issue(s);
  uint32_t acc = 0;
  for (int s = 0; s < mytiles; ++s) {
    issue(s + ST - 1);
    mbar_wait(&mb[warp][s % ST], (s / ST) & 1);
    acc ^= *reinterpret_cast<const uint32_t*>(ring + (s % ST) * 8192 + lane * 16);
    __syncwarp();
  }
  if (acc == 0x12345678) sink[0] = make_uint4(acc, 0, 0, 0);
}

static int make_map(CUtensorMap* m, void* base, size_t rows) {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return 1;
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
  cuuint64_t dims[2] = {128, rows}; cuuint64_t strides[1] = {256}; cuuint32_t box[2] = {128, 1}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  return 0;
}


__global__ void k_stream(const uint4* __restrict__ p, size_t n16, uint4* sink) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = tid; i < n16; i += nt * 8) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (i + j * nt < n16) ? __ldcs(p + i + j * nt) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc.x ^= v[j].x; acc.y ^= v[j].y; acc.z ^= v[j].z; acc.w ^= v[j].w; }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

int main(int argc, char** argv) {
  const size_t ntok = 16ull * 8 * 32776;      // C2 K cache rows
  const int nrows = 16 * 8 * 2035;             // C2 selected rows per step
  uint8_t *kc, *vc; int* idx; uint4* sink;
  CK(cudaMalloc(&kc, ntok * 512)); CK(cudaMalloc(&vc, ntok * 256));
  CK(cudaMalloc(&idx, nrows * 4)); CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(kc, 1, ntok * 256)); CK(cudaMemset(vc, 2, ntok * 256));
  std::vector<int> h(nrows);
  std::mt19937 rng(1);
  // per pair: rows drawn inside the pair's own 32776-row slab, sorted ascending (like sel)
  for (int p = 0; p < 128; ++p) {
    std::vector<int> v(2035);
    for (auto& x : v) x = p * 32776 + (rng() % 32768);
    std::sort(v.begin(), v.end());
    for (int i = 0; i < 2035; ++i) h[p * 2035 + i] = v[i];
  }
  CK(cudaMemcpy(idx, h.data(), nrows * 4, cudaMemcpyHostToDevice));
  uint8_t* flush; CK(cudaMalloc(&flush, 512 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = (double)nrows * 512;
  auto run = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemsetAsync(flush, it, 512 << 20);
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = std::min(best, ms);
    }
    printf("%-28s %8.1f us  %7.1f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    char nm[64]; snprintf(nm, 64, "ldg   grid %d x 256", blocks);
    run(nm, [&] { k_ldg<<<blocks, 256>>>((const uint4*)kc, (const uint4*)vc, idx, nrows, sink); });
  }
  CK(cudaFuncSetAttribute(k_cpas<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 3 * 8192));
  CK(cudaFuncSetAttribute(k_cpas<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4 * 8192));
  CK(cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4 * 8192));
  for (int blocks : {148 * 2, 148 * 4, 148 * 8}) {
    char nm[64];
    snprintf(nm, 64, "cpas3 grid %d x 128", blocks);
    run(nm, [&] { k_cpas<3><<<blocks, 128, 4 * 3 * 8192>>>(kc, vc, idx, nrows, sink); });
    snprintf(nm, 64, "cpas4 grid %d x 128", blocks);
    run(nm, [&] { k_cpas<4><<<blocks, 128, 4 * 4 * 8192>>>(kc, vc, idx, nrows, sink); });
    snprintf(nm, 64, "bulk4 grid %d x 128", blocks);
    run(nm, [&] { k_bulk<4><<<blocks, 128, 4 * 4 * 8192>>>(kc, vc, idx, nrows, sink); });
  }
  CK(cudaFuncSetAttribute(k_cpas<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 3 * 8192));
  {
    CUtensorMap mk, mv;
    if (!make_map(&mk, kc, ntok) && !make_map(&mv, vc, ntok)) {
      CK(cudaFuncSetAttribute(k_g4<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 3 * 8192));
      CK(cudaFuncSetAttribute(k_g4<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4 * 8192));
      for (int blocks : {148 * 2, 148 * 4}) {
        char nm[64];
        snprintf(nm, 64, "gather4 st3 %d", blocks);
        run(nm, [&] { k_g4<3><<<blocks, 128, 4 * 3 * 8192>>>(mk, mv, idx, nrows, sink); });
        snprintf(nm, 64, "gather4 st4 %d", blocks);
        run(nm, [&] { k_g4<4><<<blocks, 128, 4 * 4 * 8192>>>(mk, mv, idx, nrows, sink); });
      }
      CK(cudaGetLastError());
    }
  }
  for (int blocks : {148 * 2, 148 * 4}) {
    char nm[64];
    snprintf(nm, 64, "cpas3 interleaved %d", blocks);
    run(nm, [&] { k_cpas<3, true><<<blocks, 128, 4 * 3 * 8192>>>(kc, vc, idx, nrows, sink); });
  }
  // sequential rows (streaming ceiling of the same loader)
  std::vector<int> hs(nrows);
  for (int i = 0; i < nrows; ++i) hs[i] = i;
  CK(cudaMemcpy(idx, hs.data(), nrows * 4, cudaMemcpyHostToDevice));
  run("cpas3 sequential 296", [&] { k_cpas<3><<<296, 128, 4 * 3 * 8192>>>(kc, vc, idx, nrows, sink); });
  run("cpas3 seq interleaved 296", [&] { k_cpas<3, true><<<296, 128, 4 * 3 * 8192>>>(kc, vc, idx, nrows, sink); });
  // unsorted random rows over the whole cache
  std::mt19937 r2(7);
  for (int i = 0; i < nrows; ++i) hs[i] = r2() % (int)(ntok / 2);
  CK(cudaMemcpy(idx, hs.data(), nrows * 4, cudaMemcpyHostToDevice));
  run("cpas3 unsorted 296", [&] { k_cpas<3><<<296, 128, 4 * 3 * 8192>>>(kc, vc, idx, nrows, sink); });
  run("cpas3 unsorted interleaved 296", [&] { k_cpas<3, true><<<296, 128, 4 * 3 * 8192>>>(kc, vc, idx, nrows, sink); });
  {
    const size_t n16 = ntok * 512 / 16;  // whole kc buffer (4.3 GB)
    cudaEvent_t a0, a1; cudaEventCreate(&a0); cudaEventCreate(&a1);
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(a0); k_stream<<<blocks, 256>>>((const uint4*)kc, n16, sink); cudaEventRecord(a1);
        cudaEventSynchronize(a1); float ms; cudaEventElapsedTime(&ms, a0, a1); if (it) best = std::min(best, ms);
      }
      printf("stream-read %d x 256: %.1f GB/s\n", blocks, n16 * 16.0 / (best * 1e-3) / 1e9);
    }
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
