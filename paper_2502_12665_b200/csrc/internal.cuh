// Internal declarations shared by the kernels and the C-ABI layer.
// Product code: never includes anything from oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "a2ats.h"

namespace a2ats {

constexpr int kD = 128;     // head dimension supported by this version
constexpr int kHalf = 64;   // d / 2 rotation pairs (half-split pairing, Q2)

// Rotation frequencies theta^(-2m/d) (or the caller's override), fp64, passed by
// value to the kernels that need angles (bridge b*f_m, window r*f_m).
struct RopeTab {
  double inv_freq[kHalf];
};

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ float bf_u16(uint16_t x) { return __uint_as_float(uint32_t(x) << 16); }

// Total order on floats as unsigned keys (ascending key == ascending value); -0 is
// folded onto +0 so equal floats always get equal keys.
__device__ __forceinline__ uint32_t ordered_key(float f) {
  uint32_t u = __float_as_uint(f == 0.0f ? 0.0f : f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_nc_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- kernel argument blocks
struct LutArgs {
  const uint16_t* q;         // bf16 [B, Hq, 128]
  const uint16_t* codebook;  // bf16 [Hkv, L, 128]
  float* agg;                // [B, Hkv, L]
  float* lut_full;           // [B, Hq, L] or nullptr (debug scores)
  float* qrot;               // [B, Hq, 128]   q~ = q R_b
  float2* cs;                // [window, 64]   (cos, sin)(r f_m)
  int B, Hq, Hkv, G, L, window, bridge, group_reduce;
  RopeTab rt;
  float2 bcs[kHalf];         // (cos, sin)(b f_m), from fp64 angles on the host
};

struct SelArgs {
  const float* agg;             // [P, L]
  const int32_t* hist;          // [P, L] or nullptr
  const uint16_t* codes;        // [P, n_max]
  int32_t* sel;                 // [P, keff]
  int L, W, n_max, n_ctx, c0, c1, n_s, w0, keff;
};

struct AttnArgs {
  const uint16_t* q;      // bf16 [B, Hq, 128] pre-PE
  const float* qrot;      // [B, Hq, 128]
  const float2* cs;       // [window, 64]
  const uint16_t* kc;     // bf16 [B, Hkv, n_max, 128]
  const uint16_t* vc;
  const int32_t* sel;     // [P, keff]
  float* part;            // [P * nz, GT, nsplit, 130]
  unsigned int* counter;  // [P * nz]
  float* out;             // [B, Hq, 128]
  int Hq, Hkv, G, n_max, n_ctx, n_s, keff, n_w, w0, M, R, nsplit;
  float scale_log2;       // log2(e) / sqrt(d)
};

struct EncArgs {
  const uint16_t* keys;      // bf16 [B, Hkv, n_max, 128]
  const uint16_t* codebook;  // bf16 [Hkv, L, 128]
  const float* H;            // [Hkv, 128, 128] or nullptr
  const float* nrm;          // [Hkv, L]
  float* u;                  // ws [Hkv, vcap, 128]   u = k H
  unsigned long long* slot;  // ws [Hkv, vcap]         ~pack(dist, code), 0 = empty
  unsigned int* counter;     // ws [Hkv, vcap / 64]
  uint16_t* codes;           // [B, Hkv, n_max]
  int32_t* hist;             // [B, Hkv, L] or nullptr
  int B, Hkv, L, n_max, t_begin, T, nvec, lsplit, tiles_per_split;
};

// ---------------------------------------------------------------- launchers (return cudaError_t)
cudaError_t launch_lut(const LutArgs& a, cudaStream_t st);
cudaError_t launch_scores(const float* lut_full, const uint16_t* codes, float* scores, int B, int Hq, int Hkv,
                          int G, int L, int n_max, int n_ctx, cudaStream_t st);
cudaError_t launch_select(const SelArgs& a, int P, cudaStream_t st);
cudaError_t launch_attention(const AttnArgs& a, int P, int GT, cudaStream_t st);
cudaError_t launch_prepare(const uint16_t* codebook, const float* H, float* nrm, int Hkv, int L, cudaStream_t st);
cudaError_t launch_encode(const EncArgs& a, cudaStream_t st);

int sm_count();
int encode_codeword_tile();
int encode_key_tile();

}  // namespace a2ats
