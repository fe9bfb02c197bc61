// Micro-benchmark (tuning only, not product): HBM streaming rate of a persistent 1-CTA-per-SM
// TMA ring (1D cp.async.bulk of contiguous stages), vs ring depth / stage size / consumers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_probe tools/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  const uint32_t mm = (uint32_t)__cvta_generic_to_shared(m);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mm), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"(mm) : "memory");
}

// each CTA streams `per_cta` bytes: CTA b reads chunks b, b + grid, ... of `chunk` bytes
__global__ __launch_bounds__(128, 1) void ring_probe(const uint8_t* src, size_t total, int chunk, int stages, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[16];
  const int tid = threadIdx.x;
  const size_t nch = total / chunk;
  const size_t mine = (nch - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < stages && i < (int)mine; ++i)
      bulk(smem + (size_t)i * chunk, src + (blockIdx.x + (size_t)i * gridDim.x) * chunk, chunk, &full[i]);
  }
  __syncthreads();
  uint32_t acc = 0;
  for (size_t j = 0; j < mine; ++j) {
    const int s = j % stages;
    mbar_wait(&full[s], (uint32_t)(j / stages) & 1u);
    acc += reinterpret_cast<const uint32_t*>(smem + (size_t)s * chunk)[tid];
    __syncthreads();
    if (tid == 0 && j + stages < mine)
      bulk(smem + (size_t)s * chunk, src + (blockIdx.x + (j + stages) * gridDim.x) * chunk, chunk, &full[s]);
  }
  if (acc == 0x12345u) out[0] = acc;
}

// plain LDG.128 streaming: every thread loads 16 B per iteration, 4 loads in flight
__global__ __launch_bounds__(1024, 1) void ldg_probe(const uint4* src, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
    acc += a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) acc += __ldcs(src + i).x;
  if (acc == 0x12345u) out[0] = acc;
}

// L2 warm-up by real loads (results discarded): the first `bytes` of src
__global__ __launch_bounds__(256) void warm_probe(const uint4* src, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    acc += v.x;
  }
  if (acc == 0x12345u) out[0] = acc;
}
// bulk L2 prefetch of the first `bytes`
__global__ void pf_probe(const uint8_t* src, size_t bytes, int piece) {
  for (size_t o = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * piece; o < bytes; o += (size_t)gridDim.x * blockDim.x * piece)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + o), "r"((uint32_t)piece) : "memory");
}
__global__ void busy_probe(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}

int main() {
  const size_t total = 134217728;  // 128 MiB = the C4 codes
  uint8_t* src;
  uint32_t* out;
  cudaMalloc(&src, total);
  cudaMalloc(&out, 4);
  cudaMemset(src, 1, total);
  uint8_t* flush;
  cudaMalloc(&flush, 512u << 20);
  cudaFuncSetAttribute(ring_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  int cfg[][2] = {{32768, 2}, {32768, 4}, {32768, 6}, {16384, 4}, {16384, 8}, {16384, 12}, {8192, 8}, {8192, 16}, {65536, 3}, {16384, 13}};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& c : cfg) {
    const int chunk = c[0], stages = c[1];
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(flush, rep, 512u << 20);
      cudaEventRecord(a);
      ring_probe<<<148, 128, (size_t)chunk * stages>>>(src, total, chunk, stages, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) best = ms < best ? ms : best;
    }
    printf("chunk %6d x %2d stages (%4d KB in ring): %.2f us  %.0f GB/s  err=%s\n", chunk, stages, chunk * stages / 1024,
           best * 1e3, total / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  for (int grid : {148, 296}) {
    for (int c : {16384, 32768}) {
      const int stages = (grid == 296 ? 110 : 220) * 1024 / c;
      cudaFuncSetAttribute(ring_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaMemset(flush, rep, 512u << 20);
        cudaEventRecord(a);
        ring_probe<<<grid, 128, (size_t)c * stages>>>(src, total, c, stages, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) best = ms < best ? ms : best;
      }
      printf("grid %d chunk %d x %d: %.2f us %.0f GB/s %s\n", grid, c, stages, best * 1e3, total / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  {
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, f0;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&f0);
    for (int mode = 0; mode < 5; ++mode) {
      for (size_t warm : {32ull << 20, 64ull << 20, 96ull << 20}) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
          cudaMemset(flush, rep + 7, 512u << 20);
          cudaDeviceSynchronize();
          // s1: 20 us of busy SMs (stands for LUT + threshold), s2: warm-up concurrently; then the stream
          cudaEventRecord(f0, s1);
          cudaStreamWaitEvent(s2, f0);
          busy_probe<<<148, 128, 0, s1>>>(20000);
          if (mode == 1) warm_probe<<<148, 256, 0, s2>>>(reinterpret_cast<const uint4*>(src), warm / 16, out);
          if (mode == 2) pf_probe<<<148, 32, 0, s2>>>(src, warm, 32768);
          if (mode == 3) pf_probe<<<148, 32, 0, s2>>>(src, warm, 4096);
          if (mode == 4) warm_probe<<<74, 256, 0, s2>>>(reinterpret_cast<const uint4*>(src), warm / 16, out);
          cudaEventRecord(e1, s2);
          cudaStreamWaitEvent(s1, e1);
          cudaEventRecord(a, s1);
          ring_probe<<<148, 128, (size_t)32768 * 6, s1>>>(src, total, 32768, 6, out);
          cudaEventRecord(b, s1);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep) best = ms < best ? ms : best;
        }
        printf("mode %d (0 none, 1 ldg-warm, 2 bulk-pf 32K, 3 bulk-pf 4K, 4 ldg-warm half grid) warm %3zu MB: stream %.2f us\n", mode, warm >> 20, best * 1e3);
      }
    }
  }
  uint8_t* big;
  const size_t bigsz = 2048ull << 20;
  cudaMalloc(&big, bigsz);
  cudaMemset(big, 1, bigsz);
  for (size_t sz : {32ull << 20, 64ull << 20, 128ull << 20, 256ull << 20, 512ull << 20, 2048ull << 20}) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(flush, rep, 512u << 20);
      cudaEventRecord(a);
      ldg_probe<<<148, 1024>>>(reinterpret_cast<const uint4*>(big), sz / 16, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) best = ms < best ? ms : best;
    }
    printf("ldg %5zu MB: %.2f us %.0f GB/s\n", sz >> 20, best * 1e3, sz / (best * 1e-3) / 1e9);
  }
  for (int grid : {148, 296, 592}) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(flush, rep, 512u << 20);
      cudaEventRecord(a);
      ldg_probe<<<grid, 1024>>>(reinterpret_cast<const uint4*>(src), total / 16, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) best = ms < best ? ms : best;
    }
    printf("ldg grid %d x 1024: %.2f us %.0f GB/s %s\n", grid, best * 1e3, total / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
