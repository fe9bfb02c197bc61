// Internal declarations shared by the kernels and the C-ABI layer.
// Product code: never includes anything from oracle/.
#pragma once
#include <cuda.h>  // CUtensorMap (type only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "a2ats.h"

namespace a2ats {

constexpr int kD = 128;     // head dimension supported by this version
constexpr int kHalf = 64;   // d / 2 rotation pairs (half-split pairing, Q2)
constexpr int kMaxRanks = 8;  // sequence-sharded step: ranks of one node

// Rotation frequencies theta^(-2m/d) (or the caller's override), fp64, passed by
// value to the kernels that need angles (bridge b*f_m, window r*f_m).
struct RopeTab {
  double inv_freq[kHalf];
};

// ---------------------------------------------------------------- tuning instrumentation
// Built only into the tools/ variant (-DA2ATS_PHASES): CTA 0 of a kernel records
// clock64() at phase boundaries; each .cu exports a2ats_debug_<file>_phases().
#ifdef A2ATS_PHASES
#define A2ATS_PHASE_DECL(name) __device__ long long name[16];
#define A2ATS_PHASE(arr, i)                                                        \
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) \
    arr[i] = clock64();
#define A2ATS_PHASE_EXPORT(fn, arr)                                                           \
  extern "C" int fn(long long* out) {                                                         \
    return cudaMemcpyFromSymbol(out, arr, 16 * sizeof(long long)) == cudaSuccess ? 0 : -4; \
  }
// CTA timeline: thread 0 of every CTA records %globaltimer (ns) at its start (0)
// and end (1), optional phase marks 2..7; a2ats_debug_<kernel>_timeline() copies [kTlMax][8].
constexpr int kTlMax = 8192;
#define A2ATS_TL_DECL(name) __device__ unsigned long long name[kTlMax][8];
#define A2ATS_TL(arr, i)                                                                       \
  if (threadIdx.x == 0) {                                                                      \
    const unsigned cta_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;     \
    unsigned long long t_;                                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
    if (cta_ < kTlMax) arr[cta_][i] = t_;                                                      \
  }
// the calling thread records (the caller picks one thread)
#define A2ATS_TLX(arr, i)                                                                      \
  {                                                                                            \
    const unsigned cta_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;     \
    unsigned long long t_;                                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
    if (cta_ < kTlMax) arr[cta_][i] = t_;                                                      \
  }
// slot 7: a value (e.g. the CTA's role) instead of a time
#define A2ATS_TL_VAL(arr, v)                                                               \
  if (threadIdx.x == 0) {                                                                  \
    const unsigned cta_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; \
    if (cta_ < kTlMax) arr[cta_][7] = (unsigned long long)(v);                             \
  }
#define A2ATS_TL_EXPORT(fn, arr)                                                                        \
  extern "C" int fn(unsigned long long* out) {                                                          \
    return cudaMemcpyFromSymbol(out, arr, sizeof(unsigned long long) * 8 * a2ats::kTlMax) == cudaSuccess ? 0 : -4; \
  }
#else
#define A2ATS_PHASE_DECL(name)
#define A2ATS_PHASE(arr, i)
#define A2ATS_PHASE_EXPORT(fn, arr)
#define A2ATS_TL_DECL(name)
#define A2ATS_TL(arr, i)
#define A2ATS_TL_VAL(arr, v)
#define A2ATS_TLX(arr, i)
#define A2ATS_TL_EXPORT(fn, arr)
#endif

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the path is launched with programmatic stream serialization:
// kernel N+1 may start while kernel N runs, does its input-independent prologue
// (TMEM alloc, constant / input loads), then pdl_wait()s for N's completion.
// Each kernel calls pdl_trigger() only AFTER its own pdl_wait(), so at most two
// kernels overlap and a pre-wait prologue never races a kernel two back.  A pre-wait
// prologue reads only data written before the step or at least two launches back; a
// kernel whose output its successor reads before the wait (a2ats_stage_rows, the
// per-query-head q gather) does not trigger early, and the attention reads the window
// logits after its wait when its predecessor (a long-context / posting-list select)
// wrote them.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device (cached per
// (kernel, device) under a mutex; a second device in the same process gets its own opt-in).
cudaError_t ensure_smem_attr(const void* kernel, int bytes);
template <typename... KArgs>
inline cudaError_t ensure_smem(void (*kern)(KArgs...), int bytes) {
  return ensure_smem_attr(reinterpret_cast<const void*>(kern), bytes);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl_off = std::getenv("A2ATS_NO_PDL") != nullptr;  // debugging switch
  cfg.attrs = attr;
  cfg.numAttrs = pdl_off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

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
  uint16_t* qt;              // [Hkv, nvt, 32 chunks, NV, 8] q~ hi|lo B tiles from qprep_kernel, or nullptr
  const uint16_t* codebook;  // bf16 [Hkv, L, 128]
  float* agg;                // [B, Hkv, L]
  float* lut_full;           // [B, Hq, L] or nullptr (debug scores)
  float2* cs;                // [window, 64]   (cos, sin)(r f_m)
  int B, Hq, Hkv, G, L, window, bridge, group_reduce;
  int NV, nvt;               // query rows per MMA tile (multiple of 16, <= 256), tiles per head
  int cs_in_lut;             // 1: the persistent LUT writes the window table cs (not qprep)
  RopeTab rt;
  float2 bcs[kHalf];         // (cos, sin)(b f_m), from fp64 angles on the host
};
int lut_tile_nv(int nvec);

struct SelArgs {
  const float* agg;             // [P, L]
  int32_t* hist;                // [P, L] or nullptr (counts of the LOCAL tokens' codes)
  int append;                   // 1: token n_ctx-1 is encoded in this step: not in hist yet, code unread
  int append_hist;              // 1: select adds it to hist after taking the counts
  int hist_end;                 // hist (and the codes read) cover tokens [0, hist_end); >= w0
  const uint16_t* codes;        // [P, n_max] local code array (local index = global - shard_begin)
  const uint8_t* codes8;        // uint8 code array (code_bytes 1: posting-list select only) instead of codes
  int32_t* sel;                 // [P, sel_stride] selected global token indices, ascending
  int L, W, n_max, n_ctx, c0, c1, n_s, w0, keff, sel_stride, B;
  // sequence sharding (single GPU: shard_begin = 0, shard_len = n_max)
  int shard_begin, shard_len, rank;
  uint32_t* pinfo;              // [P, 4] key(v*), m, K_eff, E (this rank's share when sharded)
  int32_t* nsel_out;            // [P] number of locally selected tokens (sharded step)
  // long contexts (launch_select_split): per-pair class table, chunk descriptors, completion
  uint32_t* tblg;               // [P, W] compact 2-bit classes
  unsigned long long* desc;     // [P, desc_stride] published (#above, #tied) per chunk, 0 = not yet
  unsigned int* tickets;        // [2] chunk tickets handed out / CTAs finished (zero on entry and exit)
  int nchunk, desc_stride;
  int P;                        // pairs (launch_select_pipe: the scan grid is persistent)
  // sequence-sharded step with replicated histograms (a2ats_decode_step_sharded):
  // the global histogram and every rank's histogram of tokens [0, n_ctx - 1), the codes of the
  // sinks and of the most recent WR tokens (ring, slot t % WR), the ranks' global bounds
  const int32_t* hist_g;        // [P, L]
  const int32_t* hist_r;        // [world, P, L]
  const uint16_t* ring;         // [P, WR]
  const uint16_t* sinkc;        // [P, n_sink_cap]
  int WR, n_sink_cap, world, owner;
  int bounds[kMaxRanks + 1];    // rank r holds global tokens [bounds[r], bounds[r + 1])
  uint32_t* send_codes;         // [P] the new token's code (owner rank), into the all-gather message
  int sel_base;                 // added to emitted token indices (local -> global)
  // posting-list selection (a2ats_*_postings): tokens [0, n_post) grouped by code
  const int32_t* post_off;      // [P, L + 1] start of each code's list
  const int32_t* post_tok;      // [P, n_max] token indices, grouped by code
  int n_post;
  uint32_t* pbits;              // [P, pbits_stride] above / tied candidate bitmaps (bitmap path)
  int pbits_stride;
  // window logits computed by the threshold kernel before its dependency wait (long contexts;
  // otherwise the prep kernel's window role): wlog == nullptr disables
  float* wlog;                  // [P, 64, 8]
  const uint16_t* q;            // [B, Hq, 128]
  const uint16_t* kc;           // [B, Hkv, n_max, 128]
  int Hq, G, n_wl, win_lo;
  float scale_log2;
  RopeTab rt;
};

struct AttnArgs {
  const uint16_t* q;      // bf16 [B, Hq, 128] pre-PE
  const float2* cs;       // [window, 64]
  const uint16_t* kc;     // bf16 [B, Hkv, n_max, 128]
  const uint16_t* vc;
  const int32_t* sel;     // [P, sel_stride] selected global token indices, ascending
  const int32_t* nsel;    // [P] selected count per pair (sharded), or nullptr => keff
  float* part;            // [P, G, nsplit (max), 130] split partials
  unsigned int* counter;  // [P]
  float* out;             // [B, Hq, 128] normalised output (single GPU)
  float* part_out;        // [B, Hq, 130] this rank's partial (m, l, o) (sharded), or nullptr
  int Hq, Hkv, G, n_max, n_ctx, keff, sel_stride, R, nsplit;
  // rows of the Sel list held by this rank, in global token indices
  int n_s, sink_lo;       // sinks [sink_lo, sink_lo + n_s)
  int n_w, win_lo;        // window [win_lo, win_lo + n_w)
  int shard_begin;        // local row = global - shard_begin
  float scale_log2;       // log2(e) / sqrt(d)
  float2 bcs[kHalf];      // (cos, sin)(b f_m), from fp64 angles on the host
  const float* wlog;      // [P, 64, 8] logits of the first n_wl window rows (prep kernel)
  int wlog_late;          // 1: the select kernel (this grid's predecessor) writes wlog: read after the wait
  int win_as_bridge;      // 1 (standard RoPE): window rows take the bridge logit q~ . k_j like the others
  int n_wl;
};

struct EncArgs {
  const uint16_t* keys;      // bf16 [B, Hkv, n_max, 128]
  const uint16_t* chat;      // bf16 [Hkv, L, 256]   c^_j = c_j S as hi | lo
  const float* nrm;          // [Hkv, L]
  unsigned long long* slot;  // ws [Hkv, vcap]         ~pack(dist, code), 0 = empty
  unsigned int* counter;     // ws [Hkv, vcap / 64]
  uint16_t* codes;           // [B, Hkv, n_max]
  uint8_t* codes8;           // [B, Hkv, n_max] uint8 codes (code_bytes 1) instead of codes
  int32_t* hist;             // [B, Hkv, L] or nullptr
  int B, Hkv, L, n_max, t_begin, T, nvec, lsplit, tiles_per_split;
};

// ---------------------------------------------------------------- launchers (return cudaError_t)
// 2D bf16 tensor map [rows, cols] (row pitch cols * 2 B), box (64 elements, box_rows),
// SWIZZLE_128B: a box lands as the K-major SW128 layout of umma::sdesc_sw128.
cudaError_t make_tmap_sw128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);

// The step's first kernel (prep.cu): independent per-CTA roles in one launch --
//   LUT tiles (a1 + a2), decode-time encode tiles of the new keys (a0), and the
//   window rows' logits (a5's local part, Eq. 11) -- so they run concurrently.
struct PrepArgs {
  LutArgs lut;                 // LUT role (also q, rotation tables and shapes for the window role)
  EncArgs enc;                 // encode role; enc.hist == nullptr leaves the histogram to the caller
  int n_lut, n_enc, n_win;     // CTAs per role, in this order along blockIdx.x
  int lut_tx, lut_tpc, lut_cols;          // LUT: code tiles per (head, vector tile), tiles per CTA, TMEM cols
  int enc_tx, enc_tpc, enc_nv, enc_cols;  // encode: code tiles per head, tiles per CTA, keys as MMA N, TMEM cols
  // window role, one CTA per pair: logits of window tokens [win_lo, win_lo + n_wl)
  const uint16_t* kc;          // [B, Hkv, n_max, 128] (local rows: global - shard_begin)
  float* wlog;                 // [P, 64, 8] base-2 scaled logits (heads >= G: 0)
  int n_max, n_ctx, win_lo, n_wl, shard_begin;
  int win_ppc;                 // pairs per window CTA
  float scale_log2;
};
constexpr int kWinPre = 64;    // window rows per pair whose logits the prep kernel computes
int prep_lut_cols(int NV);
int prep_smem_bytes(const PrepArgs& p);  // dynamic smem of a prep launch (max over its roles)
// q~ = q R_b split hi|lo into the LUT's canonical B-tile layout (la.qt), once per step
cudaError_t launch_qprep(const LutArgs& la, cudaStream_t st);
// a2 on the FP32 pipes (lut_engine FMA / AUTO for small B*G*L): agg, lut_full and the window table
cudaError_t launch_lut_fma(const LutArgs& la, cudaStream_t st);
size_t qprep_bytes(int Hkv, int nvt, int NV);
// a2 with precomputed q~ tiles (la.qt): persistent warp-specialized tcgen05 LUT, one CTA per SM
cudaError_t launch_lut_persist(const LutArgs& la, const CUtensorMap& tm_codebook, cudaStream_t st);
cudaError_t launch_prep(const PrepArgs& p, const CUtensorMap& tm_codebook, const CUtensorMap& tm_chat,
                        cudaStream_t st);
cudaError_t launch_scores(const float* lut_full, const uint16_t* codes, float* scores, int B, int Hq, int Hkv,
                          int G, int L, int n_max, int n_ctx, cudaStream_t st);
cudaError_t launch_select(const SelArgs& a, int P, cudaStream_t st);
cudaError_t launch_select_split(const SelArgs& a, int P, cudaStream_t st);
int select_chunk_tokens();
// long-context select with hist (L <= 4096): threshold kernel (grid P) + persistent scan (nblk CTAs)
cudaError_t launch_select_pipe(const SelArgs& a, const CUtensorMap& tmK, int nblk, cudaStream_t st);
// sharded step: threshold from the replicated histograms (grid P) + the persistent scan over
// the rank's local candidate range (tmK over the local codes)
cudaError_t launch_select_shard(const SelArgs& a, const CUtensorMap& tmK, int nblk, cudaStream_t st);
// posting-list selection: one CTA per pair (threshold + bitmaps from the lists + ordered emission)
cudaError_t launch_select_postings(const SelArgs& a, cudaStream_t st);
bool select_postings_ok(int L, int n_cand);
// list-bounds row of a pair in the posting index: L + 1 int32, padded to 16 B
inline __host__ __device__ int postings_off_stride(int L) { return (L + 1 + 3) & ~3; }
inline int postings_bits_stride(int n_max) { return 2 * (((n_max + 31) / 32 + 3) & ~3); }
cudaError_t launch_postings_build(const uint16_t* codes, bool codes8, int P, int n_max, int L, int n_tok, int32_t* post_off,
                                  int32_t* post_tok, cudaStream_t st);
bool select_pipe_ok(int L);
cudaError_t launch_attention(const AttnArgs& a, int P, int GT, cudaStream_t st);
cudaError_t launch_combine(const float* parts, int R, int rows, size_t stride, float* out, cudaStream_t st);
cudaError_t launch_prepare(const uint16_t* codebook, const float* H, float* nrm, uint16_t* chat, int Hkv, int L,
                           cudaStream_t st);
cudaError_t launch_encode_bulk(const EncArgs& a, const CUtensorMap& tm_chat, cudaStream_t st);

int sm_count();
int encode_codeword_tile();
int encode_key_tile();
int encode_cw_max();  // keys per head up to which the codeword-major (decode) encoder runs

}  // namespace a2ats
