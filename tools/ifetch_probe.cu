// Instruction-fetch probe (tools only): cost of executing N instructions of cold
// straight-line code once vs. the same count from a small loop, with 128 CTAs x
// 512 threads (one CTA per SM, like the select kernel).  Prints ns per CTA (clock64 /
// 1.965 GHz nominal) for each variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ifetch_probe ifetch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define OP(i) x = x * 1664525u + (i) ; y ^= x >> 7;
#define R8(i) OP(i) OP(i + 1) OP(i + 2) OP(i + 3) OP(i + 4) OP(i + 5) OP(i + 6) OP(i + 7)
#define R64(i) R8(i) R8(i + 8) R8(i + 16) R8(i + 24) R8(i + 32) R8(i + 40) R8(i + 48) R8(i + 56)
#define R512(i) R64(i) R64(i + 64) R64(i + 128) R64(i + 192) R64(i + 256) R64(i + 320) R64(i + 384) R64(i + 448)

template <int REP>
__global__ void straight(unsigned* out, long long* cyc, unsigned seed) {
  unsigned x = seed + threadIdx.x, y = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll
  for (int r = 0; r < REP; ++r) { R512(r * 512) }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (y == 0x12345) out[0] = x;
}

__global__ void looped(unsigned* out, long long* cyc, unsigned seed, int iters) {
  unsigned x = seed + threadIdx.x, y = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < iters; ++r) { R64(r) }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (y == 0x12345) out[0] = x;
}

int main() {
  unsigned* out; long long* cyc; cudaMalloc(&out, 64); cudaMalloc(&cyc, 128 * 8);
  long long h[128];
  auto report = [&](const char* name, int ninstr) {
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0;
    for (int i = 0; i < 128; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("%-22s ~%6d src ops  mean %8.0f cyc  max %8lld cyc  (%.2f us mean)\n", name, ninstr, sum / 128.0, mx,
           sum / 128.0 / 1965.0);
  };
  for (int rep = 0; rep < 3; ++rep) {
    straight<1><<<128, 512>>>(out, cyc, rep); report("straight 512", 512);
    straight<2><<<128, 512>>>(out, cyc, rep); report("straight 1024", 1024);
    straight<4><<<128, 512>>>(out, cyc, rep); report("straight 2048", 2048);
    straight<8><<<128, 512>>>(out, cyc, rep); report("straight 4096", 4096);
    looped<<<128, 512>>>(out, cyc, rep, 8); report("loop 64 x 8", 512);
    looped<<<128, 512>>>(out, cyc, rep, 16); report("loop 64 x 16", 1024);
    looped<<<128, 512>>>(out, cyc, rep, 32); report("loop 64 x 32", 2048);
    looped<<<128, 512>>>(out, cyc, rep, 64); report("loop 64 x 64", 4096);
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
