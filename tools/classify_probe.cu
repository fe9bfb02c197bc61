// Micro-benchmark (tuning only, not product): throughput of the per-token class lookup of the
// long-context scan, codes and 32x-replicated class table in shared memory, no emission.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/classify_probe tools/classify_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

// V0: round-1 classify8s (alu-heavy)
__device__ __forceinline__ uint32_t cls_v0(uint32_t tl, uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t cls = 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t x = w[j];
    const uint32_t wl = lds_u32(((x << 3) & 0x7f80u) | tl);
    cls = __funnelshift_r(cls, __funnelshift_r(wl, wl, x << 1), 2);
    const uint32_t wh = lds_u32(((x >> 13) & 0x7f80u) | tl);
    cls = __funnelshift_r(cls, __funnelshift_r(wh, wh, x >> 15), 2);
  }
  return cls >> 16;
}
// V1: shifts on the fma pipe (IMAD.HI / IMAD), rotates + accumulate on the alu pipe
__device__ __forceinline__ uint32_t cls_v1(uint32_t tl, uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t cls = 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t x = w[j];
    const uint32_t al = ((x * 8u) & 0x7f80u) | tl;          // IMAD.SHL + LOP3
    const uint32_t ah = mulhi(x, 1u << 12) * 128u + tl;     // IMAD.HI + IMAD  (hi >> 4) * 128 + tl
    const uint32_t wl = lds_u32(al);
    const uint32_t wh = lds_u32(ah);
    cls = __funnelshift_r(cls, __funnelshift_r(wl, wl, x * 2u), 2);
    cls = __funnelshift_r(cls, __funnelshift_r(wh, wh, mulhi(x, 1u << 17)), 2);
  }
  return cls >> 16;
}
// V2: 1-bit table (hit = above or tied), word = code >> 5, bit = code & 31
__device__ __forceinline__ uint32_t cls_v2(uint32_t tl, uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t cls = 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t x = w[j];
    const uint32_t al = ((x * 4u) & 0x3f80u) | tl;
    const uint32_t ah = mulhi(x, 1u << 11) * 128u + tl;
    const uint32_t wl = lds_u32(al);
    const uint32_t wh = lds_u32(ah);
    cls = __funnelshift_r(cls, __funnelshift_r(wl, wl, x), 1);
    cls = __funnelshift_r(cls, __funnelshift_r(wh, wh, mulhi(x, 1u << 16)), 1);
  }
  return cls >> 24;
}
// V3: 2-bit, final-position rotate + LOP3 merge (no accumulate chain)
__device__ __forceinline__ uint32_t cls_v3(uint32_t tl, uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t cls = 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t x = w[j];
    const uint32_t al = ((x * 8u) & 0x7f80u) | tl;
    const uint32_t ah = mulhi(x, 1u << 12) * 128u + tl;
    const uint32_t wl = lds_u32(al);
    const uint32_t wh = lds_u32(ah);
    // field of code c at 2(c&15); move it to 4j (lo) / 4j+2 (hi)
    const uint32_t rl = __funnelshift_r(wl, wl, x * 2u - 4u * j);
    const uint32_t rh = __funnelshift_r(wh, wh, mulhi(x, 1u << 17) - (4u * j + 2u));
    cls = (cls & ~(0xfu << (4 * j))) | (rl & (3u << (4 * j))) | (rh & (0xcu << (4 * j)));
  }
  return cls;
}

// V4: V0 with 16 table replicas (lanes l and l + 16 share one: 2-way bank conflicts)
__device__ __forceinline__ uint32_t cls_v4(uint32_t tl16, uint4 v) { return cls_v0(tl16, v); }

template <int V>
__global__ __launch_bounds__(1024, 1) void probe(int iters, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t smp[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smp);
  const uint32_t tsh = (sbase + 32767u) & ~32767u;
  uint32_t* tbl = reinterpret_cast<uint32_t*>(smp + (tsh - sbase));
  uint4* codes = reinterpret_cast<uint4*>(smp + (tsh - sbase) + 32768);  // 64 KB of codes
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 8192; i += 1024) tbl[i] = 0x9e3779b9u * (i >> 5) + 0x7f4a7c15u;
  uint32_t st = 12345u + tid * 7919u;
  for (int i = tid; i < 4096; i += 1024) {
    uint4 v;
    st = st * 1664525u + 1013904223u; v.x = (st >> 20) | ((st >> 4) & 0xfff) << 16;
    st = st * 1664525u + 1013904223u; v.y = (st >> 20) | ((st >> 4) & 0xfff) << 16;
    st = st * 1664525u + 1013904223u; v.z = (st >> 20) | ((st >> 4) & 0xfff) << 16;
    st = st * 1664525u + 1013904223u; v.w = (st >> 20) | ((st >> 4) & 0xfff) << 16;
    codes[i] = v;
  }
  __syncthreads();
  const uint32_t tl = V == 4 ? (tsh | ((lane & 15) * 4u)) : (tsh | (lane * 4u));
  const uint32_t cb = (uint32_t)__cvta_generic_to_shared(codes);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t base = cb + ((tid * 4 + it * 388) & 4095) * 16;
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[q].x), "=r"(v[q].y), "=r"(v[q].z), "=r"(v[q].w) : "r"(base + ((q ^ (tid & 3)) << 4)));
    uint32_t c0, c1;
    if (V == 0) { c0 = cls_v0(tl, v[0]) | cls_v0(tl, v[1]) << 16; c1 = cls_v0(tl, v[2]) | cls_v0(tl, v[3]) << 16; }
    if (V == 1) { c0 = cls_v1(tl, v[0]) | cls_v1(tl, v[1]) << 16; c1 = cls_v1(tl, v[2]) | cls_v1(tl, v[3]) << 16; }
    if (V == 2) { c0 = cls_v2(tl, v[0]) | cls_v2(tl, v[1]) << 8 | cls_v2(tl, v[2]) << 16 | cls_v2(tl, v[3]) << 24; c1 = 0; }
    if (V == 3) { c0 = cls_v3(tl, v[0]) | cls_v3(tl, v[1]) << 16; c1 = cls_v3(tl, v[2]) | cls_v3(tl, v[3]) << 16; }
    if (V == 4) { c0 = cls_v4(tl, v[0]) | cls_v4(tl, v[1]) << 16; c1 = cls_v4(tl, v[2]) | cls_v4(tl, v[3]) << 16; }
    acc += __popc(c0 & 0x55555555u) + (__popc(c1 & 0xaaaaaaaau) << 16);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int V>
void run(const char* name) {
  const int smem = 32768 + 32768 + 65536;
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint32_t* out;
  cudaMalloc(&out, 4);
  const int iters = 2048;
  probe<V><<<148, 1024, smem>>>(16, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<V><<<148, 1024, smem>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double codes = 148.0 * 1024 * iters * 32;
  const double per_s = codes / (ms * 1e-3);
  printf("%s: %.3f ms, %.1f Gcodes/s, C4 67.1M codes -> %.2f us\n", name, ms, per_s / 1e9, 67.1e6 / per_s * 1e6);
  cudaFree(out);
}

int main() {
  run<0>("v0 round-1 (alu)");
  run<1>("v1 fma-shifts  ");
  run<2>("v2 1-bit       ");
  run<3>("v3 final-pos   ");
  run<4>("v4 16 replicas ");
  return 0;
}
