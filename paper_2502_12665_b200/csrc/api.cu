// C-ABI of liba2ats.so (declared and documented in include/a2ats.h).
// Host orchestration only: validation, workspace carving, kernel launches on
// the caller's stream.  No allocation, no host synchronisation.
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "internal.cuh"

namespace a2ats {

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

cudaError_t ensure_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes opted in
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{kernel, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  // the SM's shared / L1 split is fixed while CTAs are resident: at the maximum shared carveout
  // a kernel's CTAs can join an SM that runs the previous kernel's (programmatic dependent launch)
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) have = bytes;
  return e;
}

// Tuning switches (tools/ variant builds): contexts of at least this many 32K-token code chunks
// take the threshold + persistent scan select; query tiles wider than this many vectors take
// the qprep kernel (q~ once per step instead of in every LUT CTA).
#ifndef A2ATS_PIPE_MIN_CHUNKS
#define A2ATS_PIPE_MIN_CHUNKS 2
#endif
#ifndef A2ATS_POST_WLOG
#define A2ATS_POST_WLOG 1  // tuning define: the posting select precomputes the first 64 window logits
#endif
#ifndef A2ATS_LUT_PERSIST
#define A2ATS_LUT_PERSIST 1  // persistent warp-specialized LUT for precomputed q~ tiles (tuning define)
#endif
#ifndef A2ATS_QPREP_MIN_NV
#define A2ATS_QPREP_MIN_NV 64
#endif

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Rows of the Sel list handled by one attention CTA (one 8-warp CTA per SM).  Fixed
// per (shape, params) -- not per n_ctx -- so the workspace size is too: with enough
// (b, KV head) pairs to fill the GPU a pair is one CTA (no cross-CTA combine) up to
// kAttnRowsMax rows; with few pairs the rows are split so the grid covers the SMs.
constexpr int kAttnRowsMax = 2048;  // s_tok capacity of the attention smem layout
#ifndef A2ATS_ATTN_SPLITS
#define A2ATS_ATTN_SPLITS 0  // tuning builds only: force the splits per pair (0 = heuristic below)
#endif
int attn_rows(int P, long long mmax) {
  const int sms = sm_count();
  long long want = (4LL * P >= 3LL * sms) ? 1 : (sms + P - 1) / P;  // splits per pair
  if (A2ATS_ATTN_SPLITS > 0) want = A2ATS_ATTN_SPLITS;
  long long R = (mmax + want - 1) / want;
  R = (R + 15) / 16 * 16;
  return (int)std::max<long long>(256, std::min<long long>(kAttnRowsMax, R));
}
long long attn_mmax(const a2ats_shape* s, const a2ats_params* p) {
  return std::min<long long>(p->topk, s->n_max) + p->n_sink + p->window;
}

struct Derived {
  int G, P, n_w, w0, n_s, c0, c1, n_cand, keff, M;
  int R, nsplit, GT, nz, W;
};

int check_shape(const a2ats_shape* s) {
  if (!s) return A2ATS_EINVAL;
  if (s->B <= 0 || s->Hq <= 0 || s->Hkv <= 0 || s->d <= 0 || s->L <= 0 || s->n_max <= 0) return A2ATS_EINVAL;
  if (s->d % 2) return A2ATS_EINVAL;
  if (s->Hq % s->Hkv) return A2ATS_EINVAL;
  if (s->n_max % 8) return A2ATS_EINVAL;
  if (s->code_bytes < 0 || s->code_bytes > 2) return A2ATS_EINVAL;
  if (s->code_bytes == 1 && s->L > 256) return A2ATS_EUNSUPPORTED;
  if (s->d != kD) return A2ATS_EUNSUPPORTED;
  const int G = s->Hq / s->Hkv;
  if (G != 1 && G != 2 && G != 4 && G != 8) return A2ATS_EUNSUPPORTED;
  if (s->L > 16384) return A2ATS_EUNSUPPORTED;
  return A2ATS_OK;
}

int check_params(const a2ats_params* p) {
  if (!p) return A2ATS_EINVAL;
  if (p->window < 1 || p->bridge < 0 || p->n_sink < 0 || p->topk < 0) return A2ATS_EINVAL;
  if (!(p->rope_theta > 0.0) && !p->inv_freq) return A2ATS_EINVAL;
  if (p->group_reduce != A2ATS_GROUP_MAX && p->group_reduce != A2ATS_GROUP_SUM &&
      p->group_reduce != A2ATS_GROUP_PER_HEAD)
    return A2ATS_EINVAL;
  if (p->kv_location != A2ATS_KV_DEVICE && p->kv_location != A2ATS_KV_HOST_MAPPED) return A2ATS_EINVAL;
  if (p->lut_engine < A2ATS_LUT_AUTO || p->lut_engine > A2ATS_LUT_FMA) return A2ATS_EINVAL;
  if (p->hist_lag < 0 || p->hist_lag > p->window) return A2ATS_EINVAL;
  if (p->rope_mode != A2ATS_ROPE_WINDOWED && p->rope_mode != A2ATS_ROPE_STANDARD) return A2ATS_EINVAL;
  return A2ATS_OK;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

void derive(const a2ats_shape* s, const a2ats_params* p, int n_ctx, Derived* d) {
  d->G = s->Hq / s->Hkv;
  d->P = s->B * s->Hkv;
  d->n_w = std::min(p->window, n_ctx);              // W = {t >= N - w}     (Eq. 11 locality)
  d->w0 = n_ctx - d->n_w;
  d->n_s = std::min(p->n_sink, d->w0);              // sinks outside W
  d->c0 = d->n_s;
  d->c1 = d->w0;
  d->n_cand = d->c1 - d->c0;
  d->keff = std::min(p->topk, d->n_cand);
  d->M = d->n_s + d->keff + d->n_w;
  d->R = attn_rows(d->P, attn_mmax(s, p));
  d->nsplit = (d->M + d->R - 1) / d->R;
  d->GT = d->G >= 4 ? 4 : d->G;
  d->nz = d->G / d->GT;
  d->W = (s->L + 15) / 16;
}

struct DecodeWs {
  size_t cs, agg, lut, sel, part, actr, pinfo, nsel, wlog, eslot, ectr, tblg, desc, tick, qt, pbits, total;
};

DecodeWs decode_layout(const a2ats_shape* s, const a2ats_params* p) {
  const int G = s->Hq / s->Hkv, P = s->B * s->Hkv;
  const long long kmax = std::min<long long>(p->topk, s->n_max);
  const long long mmax = attn_mmax(s, p);
  const int R = attn_rows(P, mmax);
  const long long nsplit_max = (mmax + R - 1) / R;
  const int GT = G >= 4 ? 4 : G;
  DecodeWs w;
  size_t o = 0;
  // regions that must be zero on entry (each kernel leaves them zero on exit) come first, at
  // offsets that depend on the shape only: params (topk, window) may change between calls on
  // the same workspace without moving them onto bytes other regions left non-zero
  w.actr = o; o = align_up(o + (size_t)P * (G / GT) * 4);                                    // attention split counters
  w.eslot = o; o = align_up(o + (size_t)s->Hkv * std::max(s->B, 1) * 8);                    // append encode slots
  w.ectr = o; o = align_up(o + (size_t)s->Hkv * 2 * 4);
  w.desc = o; o = align_up(o + (size_t)P * (s->n_max / select_chunk_tokens() + 2) * 8);     // look-back descriptors
  w.tick = o; o = align_up(o + 8);                                                           // chunk tickets
  w.cs = o; o = align_up(o + (size_t)p->window * kHalf * 8);
  w.agg = o; o = align_up(o + (size_t)P * s->L * 4);
  w.lut = o; o = align_up(o + (size_t)s->B * s->Hq * s->L * 4);
  w.sel = o; o = align_up(o + (size_t)P * std::max<long long>(kmax, 1) * 4);
  w.part = o; o = align_up(o + (size_t)P * (G / GT) * GT * nsplit_max * 130 * 4);
  w.pinfo = o; o = align_up(o + (size_t)P * 16);
  w.nsel = o; o = align_up(o + (size_t)P * 4);
  w.wlog = o; o = align_up(o + (size_t)P * kWinPre * 8 * 4);
  w.tblg = o; o = align_up(o + (size_t)P * ((s->L + 15) / 16) * 4);                       // long-context select
  {
    const int NV = lut_tile_nv(s->B * G), nvt = (s->B * G + NV - 1) / NV;
    w.qt = o; o = align_up(o + qprep_bytes(s->Hkv, nvt, NV));                                // q~ B tiles
  }
  w.pbits = o; o = align_up(o + (size_t)P * postings_bits_stride(s->n_max) * 4);             // postings bitmap path
  w.total = o;
  return w;
}

// Per-query-head selection (A2ATS_GROUP_PER_HEAD, G > 1): G sub-steps on the shape with Hq' = Hkv
// (G' = 1); the workspace holds the sub-step's own layout first, then q of one head position g
// [B, Hkv, d] bf16, the sub-step's output [B, Hkv, d] fp32 and selection [B, Hkv, K] int32.
bool per_head(const a2ats_shape* s, const a2ats_params* p) {
  return p->group_reduce == A2ATS_GROUP_PER_HEAD && s->Hq != s->Hkv;
}
struct PerHeadWs {
  a2ats_shape sub;
  a2ats_params subp;
  size_t inner, qg, outg, selg, total;
};
PerHeadWs per_head_layout(const a2ats_shape* s, const a2ats_params* p) {
  PerHeadWs w;
  w.sub = *s;
  w.sub.Hq = s->Hkv;
  w.subp = *p;
  w.subp.group_reduce = A2ATS_GROUP_MAX;  // (one query head per group: the fold is the identity)
  const size_t P = (size_t)s->B * s->Hkv;
  size_t o = 0;
  w.inner = o; o = align_up(o + decode_layout(&w.sub, &w.subp).total);
  w.qg = o; o = align_up(o + P * kD * 2);
  w.outg = o; o = align_up(o + P * kD * 4);
  w.selg = o; o = align_up(o + P * (size_t)std::max<long long>(std::min<long long>(p->topk, s->n_max), 1) * 4);
  w.total = o;
  return w;
}

constexpr int kEncVcap = 16384;  // key vectors per KV head encoded per launch

struct EncodeWs {
  size_t slot, ctr, total;
};
EncodeWs encode_layout(const a2ats_shape* s) {
  EncodeWs w;
  size_t o = 0;
  w.slot = o; o = align_up(o + (size_t)s->Hkv * kEncVcap * 8);
  w.ctr = o; o = align_up(o + (size_t)s->Hkv * (kEncVcap / 64) * 4);
  w.total = o;
  return w;
}

struct PostingsLayout {
  size_t off, tok, total;
};
PostingsLayout postings_layout(const a2ats_shape* s) {
  PostingsLayout w;
  const size_t P = (size_t)s->B * s->Hkv;
  w.off = 0;
  w.tok = align_up(P * postings_off_stride(s->L) * 4);
  w.total = align_up(w.tok + P * s->n_max * 4);
  return w;
}

void fill_rope(const a2ats_params* p, RopeTab* rt) {
  for (int m = 0; m < kHalf; ++m)
    rt->inv_freq[m] = p->inv_freq ? p->inv_freq[m] : std::pow(p->rope_theta, -2.0 * m / (double)kD);
}

// bridge rotation R_b: fp64 angles b f_m, fp32 (cos, sin) (reading Q16)
void fill_bcs(const a2ats_params* p, const RopeTab& rt, float2* bcs) {
  for (int m = 0; m < kHalf; ++m) {
    const double ang = (double)p->bridge * rt.inv_freq[m];
    bcs[m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
}

}  // namespace

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t make_tmap_sw128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// codes [P, n_max] u16 viewed as [P][n_max / 64][64] (128-B rows), box = 256 rows of one pair,
// SWIZZLE_128B (n_max % 64 == 0): the long-context select's stage loads
cudaError_t make_tmap_codes(CUtensorMap* map, const void* codes, uint64_t P, uint64_t n_max) {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[3] = {64, n_max / 64, P};
  const cuuint64_t strides[2] = {128, n_max * 2};
  const cuuint32_t box[3] = {64, 256, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(codes), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

namespace {
// last CUDA failure (code + api.cu line of the launch), for a2ats_last_cuda_error()
thread_local char g_last_err[160] = "";
inline int cuda_status(cudaError_t e, int line = __builtin_LINE()) {
  if (e == cudaSuccess) return A2ATS_OK;
  std::snprintf(g_last_err, sizeof(g_last_err), "%s (%s) at api.cu:%d", cudaGetErrorName(e), cudaGetErrorString(e),
                line);
  return A2ATS_ECUDA;
}

// Benchmark instrumentation (a2ats_set_stage_events).
constexpr int kStageEvents = 5;
bool g_stage_on = false;
cudaEvent_t g_stage[kStageEvents];
inline void stage_mark(int i, cudaStream_t st) {
  if (g_stage_on) cudaEventRecord(g_stage[i], st);
}

LutArgs make_lut_args(const a2ats_shape* shape, const a2ats_params* params, const Derived& d, const void* q,
                      const void* codebook, float* agg, float* lut_full, float2* cs) {
  LutArgs la;
  la.cs_in_lut = 0;
  la.q = static_cast<const uint16_t*>(q);
  la.qt = nullptr;
  la.codebook = static_cast<const uint16_t*>(codebook);
  la.agg = agg;
  la.lut_full = lut_full;
  la.cs = cs;
  la.B = shape->B;
  la.Hq = shape->Hq;
  la.Hkv = shape->Hkv;
  la.G = d.G;
  la.L = shape->L;
  la.window = params->window;
  la.bridge = params->bridge;
  la.group_reduce = params->group_reduce;
  la.NV = lut_tile_nv(shape->B * d.G);
  la.nvt = (shape->B * d.G + la.NV - 1) / la.NV;
  fill_rope(params, &la.rt);
  fill_bcs(params, la.rt, la.bcs);
  return la;
}

constexpr float kScaleLog2 = (float)(1.4426950408889634 / 11.313708498984761);  // log2(e) / sqrt(128)

// prep kernel roles: LUT over every (code tile, vector tile, head)
void prep_set_lut(PrepArgs& p, const LutArgs& la, int tpc = 1) {
  p.lut = la;
  p.lut_tx = (la.L + 127) / 128;
  p.lut_tpc = tpc;
  p.n_lut = (p.lut_tx + tpc - 1) / tpc * la.nvt * la.Hkv;
  p.lut_cols = prep_lut_cols(la.NV);
}
// window logits of tokens [win_lo, win_lo + min(n_w, 64)) of every pair
void prep_set_window(PrepArgs& p, const a2ats_shape* s, const void* k_cache, float* wlog, int n_ctx, int win_lo,
                     int n_w, int shard_begin) {
  p.kc = static_cast<const uint16_t*>(k_cache);
  p.wlog = wlog;
  p.n_max = s->n_max;
  p.n_ctx = n_ctx;
  p.win_lo = win_lo;
  p.n_wl = std::max(0, std::min(n_w, kWinPre));
  p.shard_begin = shard_begin;
  p.scale_log2 = kScaleLog2;
  p.win_ppc = std::max(p.win_ppc, 1);
  p.n_win = p.n_wl > 0 ? (s->B * s->Hkv + p.win_ppc - 1) / p.win_ppc : 0;
}
// decode-time encode of tokens [t_begin, t_begin + T) (B * T <= encode_cw_max() keys per head)
void prep_set_encode(PrepArgs& p, const EncArgs& e, int tpc = 1) {
  p.enc = e;
  p.enc_tx = (e.L + 127) / 128;
  p.enc_tpc = tpc;
  p.n_enc = (p.enc_tx + tpc - 1) / tpc * e.Hkv;
  p.enc_nv = (e.nvec + 15) / 16 * 16;
  p.enc_cols = prep_lut_cols(p.enc_nv);
}
// Code tiles per CTA for the LUT / encode roles so that all prep CTAs are resident at once
// (one wave: the roles then run concurrently), doubling the encode's first.
#ifndef A2ATS_PREP_WAVES
#define A2ATS_PREP_WAVES 1
#endif
void prep_balance(PrepArgs& p) {
  const int per_sm = std::max(1, (227 * 1024) / (prep_smem_bytes(p) + 1024));
  const int cap = A2ATS_PREP_WAVES * per_sm * sm_count();
  const int npairs = p.lut.B * p.lut.Hkv;
  for (int guard = 0; guard < 24 && p.n_lut + p.n_enc + p.n_win > cap; ++guard) {
    // shrink the role with the most CTAs per unit of work first
    if (p.n_win && p.n_win >= p.n_lut && p.n_win >= p.n_enc && p.win_ppc < npairs) {
      p.win_ppc *= 2;
      p.n_win = (npairs + p.win_ppc - 1) / p.win_ppc;
    } else if (p.n_enc && p.n_enc >= p.n_lut && p.enc_tpc < p.enc_tx) {
      prep_set_encode(p, p.enc, p.enc_tpc * 2);
    } else if (p.n_lut && p.lut_tpc < p.lut_tx) {
      prep_set_lut(p, p.lut, p.lut_tpc * 2);
    } else if (p.n_enc && p.enc_tpc < p.enc_tx) {
      prep_set_encode(p, p.enc, p.enc_tpc * 2);
    } else if (p.n_win && p.win_ppc < npairs) {
      p.win_ppc *= 2;
      p.n_win = (npairs + p.win_ppc - 1) / p.win_ppc;
    } else {
      break;
    }
  }
}

PrepArgs prep_empty() {
  PrepArgs p;
  std::memset(&p, 0, sizeof(p));
  p.lut_tpc = p.enc_tpc = p.win_ppc = 1;
  return p;
}

}  // namespace
}  // namespace a2ats

using namespace a2ats;

extern "C" {

void a2ats_default_params(a2ats_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->window = 64;
  p->bridge = 2048;
  p->n_sink = 4;
  p->topk = 0;
  p->rope_theta = 1e4;
  p->inv_freq = nullptr;
  p->group_reduce = A2ATS_GROUP_MAX;
  p->kv_location = A2ATS_KV_DEVICE;
  p->lut_engine = A2ATS_LUT_AUTO;
}

const char* a2ats_status_string(int status) {
  switch (status) {
    case A2ATS_OK: return "A2ATS_OK";
    case A2ATS_EINVAL: return "A2ATS_EINVAL: invalid argument";
    case A2ATS_EUNSUPPORTED: return "A2ATS_EUNSUPPORTED: shape not supported by this build";
    case A2ATS_EWORKSPACE: return "A2ATS_EWORKSPACE: workspace missing or too small";
    case A2ATS_ECUDA: return "A2ATS_ECUDA: CUDA launch failed";
    case A2ATS_ENCCL: return "A2ATS_ENCCL: NCCL call failed";
    default: return "A2ATS: unknown status";
  }
}

int a2ats_abi_version(void) { return A2ATS_ABI_VERSION; }

const char* a2ats_last_cuda_error(void) { return g_last_err; }

int a2ats_set_stage_events(void* const* events, int n) {
  if (!events) {
    g_stage_on = false;
    return A2ATS_OK;
  }
  if (n < kStageEvents) return A2ATS_EINVAL;
  for (int i = 0; i < kStageEvents; ++i) {
    if (!events[i]) return A2ATS_EINVAL;
    g_stage[i] = static_cast<cudaEvent_t>(events[i]);
  }
  g_stage_on = true;
  return A2ATS_OK;
}

int a2ats_qavq_prepare(const a2ats_shape* shape, const void* codebook, const float* H, float* nrm, void* chat,
                       void* stream) {
  int rc = check_shape(shape);
  if (rc) return rc;
  if (!codebook || !nrm || !chat || !aligned16(codebook) || !aligned16(chat) || (H && !aligned16(H)))
    return A2ATS_EINVAL;
  return cuda_status(launch_prepare(static_cast<const uint16_t*>(codebook), H, nrm, static_cast<uint16_t*>(chat),
                                    shape->Hkv, shape->L, static_cast<cudaStream_t>(stream)));
}

size_t a2ats_build_codes_workspace_bytes(const a2ats_shape* shape) {
  if (check_shape(shape)) return 0;
  return encode_layout(shape).total;
}

int a2ats_build_codes(const a2ats_shape* shape, const void* keys, int32_t t_begin, int32_t t_end,
                      const void* chat, const float* nrm, uint16_t* codes, int32_t* hist, void* ws,
                      size_t ws_bytes, void* stream) {
  int rc = check_shape(shape);
  if (rc) return rc;
  if (!keys || !chat || !nrm || !codes) return A2ATS_EINVAL;
  if (!aligned16(keys) || !aligned16(chat)) return A2ATS_EINVAL;
  if (t_begin < 0 || t_end < t_begin || t_end > shape->n_max) return A2ATS_EINVAL;
  const EncodeWs L = encode_layout(shape);
  if (!ws || ws_bytes < L.total) return A2ATS_EWORKSPACE;
  if (t_end == t_begin) return A2ATS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  EncArgs a;
  a.keys = static_cast<const uint16_t*>(keys);
  a.chat = static_cast<const uint16_t*>(chat);
  a.nrm = nrm;
  a.slot = reinterpret_cast<unsigned long long*>(base + L.slot);
  a.counter = reinterpret_cast<unsigned int*>(base + L.ctr);
  a.codes = shape->code_bytes == 1 ? nullptr : codes;
  a.codes8 = shape->code_bytes == 1 ? reinterpret_cast<uint8_t*>(codes) : nullptr;
  a.hist = hist;
  a.B = shape->B;
  a.Hkv = shape->Hkv;
  a.L = shape->L;
  a.n_max = shape->n_max;
  CUtensorMap tm;
  rc = cuda_status(make_tmap_sw128(&tm, chat, (uint64_t)shape->Hkv * shape->L, 2 * kD, encode_codeword_tile()));
  if (rc) return rc;
  const int ntiles = (shape->L + encode_codeword_tile() - 1) / encode_codeword_tile();
  const int tmax = std::max(1, kEncVcap / shape->B);  // tokens per launch so that B*T <= vcap
  for (int t0 = t_begin; t0 < t_end; t0 += tmax) {
    a.t_begin = t0;
    a.T = std::min(tmax, t_end - t0);
    a.nvec = shape->B * a.T;
    if (a.nvec > kEncVcap) return A2ATS_EUNSUPPORTED;  // B > vcap
    const int vt = (a.nvec + encode_key_tile() - 1) / encode_key_tile();
    // split the codeword range so the grid covers the machine about twice
    int lsplit = (2 * sm_count() + vt * shape->Hkv - 1) / (vt * shape->Hkv);
    lsplit = std::max(1, std::min(lsplit, ntiles));
    a.tiles_per_split = (ntiles + lsplit - 1) / lsplit;
    a.lsplit = (ntiles + a.tiles_per_split - 1) / a.tiles_per_split;
    if (a.nvec <= encode_cw_max()) {
      PrepArgs p = prep_empty();
      prep_set_encode(p, a);
      rc = cuda_status(launch_prep(p, tm, tm, st));
    } else {
      rc = cuda_status(launch_encode_bulk(a, tm, st));
    }
    if (rc) return rc;
  }
  return A2ATS_OK;
}

size_t a2ats_decode_workspace_bytes(const a2ats_shape* shape, const a2ats_params* params) {
  if (check_shape(shape) || check_params(params)) return 0;
  return per_head(shape, params) ? per_head_layout(shape, params).total : decode_layout(shape, params).total;
}

}  // extern "C"

namespace a2ats {
namespace {
// Per-query-head selection plumbing (no arithmetic): q of head position g -> [B, Hkv, d]; the
// sub-step's output rows and selection rows back to (b, h * G + g).  One 16-B piece per thread.
__global__ __launch_bounds__(256) void head_gather_q_kernel(const uint4* q, uint4* qg, int P, int Hkv, int G, int g) {
  pdl_wait();  // the previous sub-step reads qg
  // no early pdl_trigger(): the sub-step's kernels read q (= qg) in their pre-wait prologues, so
  // they launch only at this grid's completion (implicit trigger), as after a2ats_stage_rows

  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * 16) return;
  const int r = i >> 4, b = r / Hkv, h = r - b * Hkv;
  qg[i] = q[((size_t)b * Hkv * G + (size_t)h * G + g) * 16 + (i & 15)];
}
__global__ __launch_bounds__(256) void head_scatter_kernel(const uint4* outg, uint4* out, const int32_t* selg,
                                                           int32_t* sel, int P, int Hkv, int G, int g, int keff) {
  pdl_wait();  // the sub-step's attention / select wrote outg, selg
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (out && i < P * 32) {
    const int r = i >> 5, b = r / Hkv, h = r - b * Hkv;
    out[((size_t)b * Hkv * G + (size_t)h * G + g) * 32 + (i & 31)] = outg[i];
  }
  if (sel) {
    for (long long j = i; j < (long long)P * keff; j += (long long)gridDim.x * blockDim.x) {
      const int r = (int)(j / keff), b = r / Hkv, h = r - b * Hkv;
      sel[((size_t)b * Hkv * G + (size_t)h * G + g) * keff + (j - (long long)r * keff)] = selg[j];
    }
  }
}
}  // namespace
}  // namespace a2ats

namespace {
int decode_impl_one(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                    const void* k_cache, const void* v_cache, uint16_t* codes, const void* codebook, int32_t* hist,
                    const void* chat, const float* nrm, float* out, int32_t* sel_out, float* scores_out, void* ws,
                    size_t ws_bytes, void* stream, bool attend, const void* postings, int32_t n_post);

// One decode step (a1..a6); with chat != nullptr also a0 for token n_ctx - 1 (append).  Per-query-
// head selection (A2ATS_GROUP_PER_HEAD, G > 1): G sub-steps with G' = 1, the append (a0 + hist) in
// the first only.
int decode_impl(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                const void* k_cache, const void* v_cache, uint16_t* codes, const void* codebook, int32_t* hist,
                const void* chat, const float* nrm, float* out, int32_t* sel_out, float* scores_out, void* ws,
                size_t ws_bytes, void* stream, bool attend = true, const void* postings = nullptr,
                int32_t n_post = 0) {
  int rc = check_shape(shape);
  if (rc) return rc;
  rc = check_params(params);
  if (rc) return rc;
  if (!per_head(shape, params)) {
    a2ats_params p1 = *params;
    if (p1.group_reduce == A2ATS_GROUP_PER_HEAD) p1.group_reduce = A2ATS_GROUP_MAX;  // (G = 1)
    return decode_impl_one(shape, &p1, n_ctx, q, k_cache, v_cache, codes, codebook, hist, chat, nrm, out, sel_out,
                           scores_out, ws, ws_bytes, stream, attend, postings, n_post);
  }
  if (scores_out) return A2ATS_EUNSUPPORTED;
  if (!q || !aligned16(q) || n_ctx <= 0 || n_ctx > shape->n_max) return A2ATS_EINVAL;
  if (attend ? !out : !sel_out) return A2ATS_EINVAL;
  const PerHeadWs L = per_head_layout(shape, params);
  if (!ws || ws_bytes < L.total) return A2ATS_EWORKSPACE;
  Derived d;
  derive(&L.sub, &L.subp, n_ctx, &d);
  const int G = shape->Hq / shape->Hkv, P = shape->B * shape->Hkv;
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint4* qg = reinterpret_cast<uint4*>(base + L.qg);
  float* outg = reinterpret_cast<float*>(base + L.outg);
  int32_t* selg = reinterpret_cast<int32_t*>(base + L.selg);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int g = 0; g < G; ++g) {
    rc = cuda_status(launch_pdl(head_gather_q_kernel, dim3((P * 16 + 255) / 256), dim3(256), 0, st,
                                static_cast<const uint4*>(q), qg, P, shape->Hkv, G, g));
    if (rc) return rc;
    rc = decode_impl_one(&L.sub, &L.subp, n_ctx, qg, k_cache, v_cache, codes, codebook, hist,
                         g == 0 ? chat : nullptr, g == 0 ? nrm : nullptr, attend ? outg : nullptr,
                         (sel_out || !attend) ? selg : nullptr, nullptr, base + L.inner, L.qg - L.inner, stream,
                         attend, postings, n_post);
    if (rc) return rc;
    const int keff = sel_out ? d.keff : 0;
    const long long work = std::max<long long>((long long)P * 32, (long long)P * keff);
    const int grid = (int)std::min<long long>((work + 255) / 256, 4096);
    rc = cuda_status(launch_pdl(head_scatter_kernel, dim3(std::max(grid, 1)), dim3(256), 0, st,
                                reinterpret_cast<const uint4*>(outg), attend ? reinterpret_cast<uint4*>(out) : nullptr,
                                selg, sel_out, P, shape->Hkv, G, g, keff));
    if (rc) return rc;
  }
  return A2ATS_OK;
}

// One decode step (a1..a6) of one selection mode (max / sum fold, or G = 1).
int decode_impl_one(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                    const void* k_cache, const void* v_cache, uint16_t* codes, const void* codebook, int32_t* hist,
                const void* chat, const float* nrm, float* out, int32_t* sel_out, float* scores_out, void* ws,
                size_t ws_bytes, void* stream, bool attend, const void* postings, int32_t n_post) {
  int rc = check_shape(shape);
  if (rc) return rc;
  rc = check_params(params);
  if (rc) return rc;
  // standard RoPE (ablation baseline): q~ = q R_{N-1}, the bridge of every row; no per-row rotation
  const bool rope_std = params->rope_mode == A2ATS_ROPE_STANDARD;
  a2ats_params pstd;
  if (rope_std) {
    if (n_ctx <= 0) return A2ATS_EINVAL;
    pstd = *params;
    pstd.bridge = n_ctx - 1;
    params = &pstd;
  }
  if (attend) {
    if (!k_cache || !v_cache || !out || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out))
      return A2ATS_EINVAL;
  } else if (!sel_out || chat) {
    return A2ATS_EINVAL;
  }
  if (!q || !codes || !codebook || !aligned16(q) || !aligned16(codes) || !aligned16(codebook)) return A2ATS_EINVAL;
  if (n_ctx <= 0 || n_ctx > shape->n_max) return A2ATS_EINVAL;
  const bool append = chat != nullptr;
  if (append && (!nrm || !aligned16(chat) || shape->B > encode_cw_max() ||
                 params->kv_location != A2ATS_KV_DEVICE))
    return A2ATS_EINVAL;
  const DecodeWs Lw = decode_layout(shape, params);
  if (!ws || ws_bytes < Lw.total) return A2ATS_EWORKSPACE;

  Derived d;
  derive(shape, params, n_ctx, &d);
  // deferred a0: the newest hist_lag tokens are in the window (never candidates); not with append
  if (params->hist_lag > d.n_w || (params->hist_lag && (append || scores_out))) return A2ATS_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  float2* cs = reinterpret_cast<float2*>(base + Lw.cs);
  float* agg = reinterpret_cast<float*>(base + Lw.agg);
  float* lut_full = scores_out ? reinterpret_cast<float*>(base + Lw.lut) : nullptr;
  float* wlog = reinterpret_cast<float*>(base + Lw.wlog);
  int32_t* sel = sel_out ? sel_out : reinterpret_cast<int32_t*>(base + Lw.sel);

  // prep: a1 + a2 (LUT), the window rows' logits and (append) a0 for token n_ctx - 1, as
  // concurrent roles of one kernel; the new token is inside the window, so the selection never
  // reads its code, and its histogram entry is added by the select kernel after its counts
  LutArgs la = make_lut_args(shape, params, d, q, codebook, agg, lut_full, cs);
  // LUT engine (a2): FP32 FMA for small B*G*L, tensor cores otherwise (reading of SURVEY 8d C5)
  const bool lut_fma = params->lut_engine == A2ATS_LUT_FMA ||
                       (params->lut_engine == A2ATS_LUT_AUTO && shape->B * d.G <= A2ATS_LUT_FMA_MAX_VECTORS);
  // wide query tiles: q~ hi|lo computed once by qprep_kernel instead of in every LUT CTA
  if (la.NV > A2ATS_QPREP_MIN_NV && !lut_fma) la.qt = reinterpret_cast<uint16_t*>(base + Lw.qt);
  PrepArgs p = prep_empty();
  prep_set_lut(p, la);
  // lut_fma_kernel (FMA engine) or lut_persist_kernel (precomputed q~ tiles) computes agg before
  // the prep kernel, which then runs only its encode / window roles
  const bool lut_persist = la.qt != nullptr && A2ATS_LUT_PERSIST;
  la.cs_in_lut = lut_persist ? 1 : 0;
  if (lut_fma || lut_persist) p.n_lut = 0;
  // long contexts: the window logits are computed by the select threshold kernel, before its
  // dependency wait (it waits for this kernel anyway); otherwise by the prep kernel's window role
  const int nchunk = d.c1 > d.c0 ? (d.c1 - ((d.c0 >> 3) << 3) + select_chunk_tokens() - 1) / select_chunk_tokens() : 0;
  const bool long_select = d.keff > 0 && nchunk >= A2ATS_PIPE_MIN_CHUNKS;
  // hist given: the warp-specialized persistent select (forward / backward half per pair);
  // otherwise threshold + chunked scan (the counts need a pass over the codes)
  // posting lists given: one CTA per pair reads only the hit codes' lists (f3)
  // (uint8 codes: the posting-list kernel is the only reader, also for the append's histogram)
  const bool post_select = postings != nullptr && (d.keff > 0 || shape->code_bytes == 1);
  if (shape->code_bytes == 1 && (postings == nullptr || scores_out)) return A2ATS_EUNSUPPORTED;
  const bool pipe_select = !post_select && long_select && hist != nullptr && select_pipe_ok(shape->L) &&
                           shape->n_max % 64 == 0;
  const bool split_select = !post_select && long_select && !pipe_select;
  prep_set_window(p, shape, k_cache, wlog, n_ctx, d.w0, d.n_w, 0);
  // posting-list select (A2ATS_POST_WLOG 0): no window logits precomputed -- the attention rotates
  // every window row itself (its cs-table branch), the select keeps its small shared memory
  const int n_wl = ((post_select && !A2ATS_POST_WLOG) || rope_std) ? 0 : p.n_wl;
  if (rope_std) p.n_win = 0;  // (no window-row logits: every row takes the bridge logit)
  // long contexts / postings: the threshold (postings) kernel computes the window logits before its wait
  if (long_select || post_select || !attend) p.n_win = 0;
  CUtensorMap tmA, tmC;
  rc = cuda_status(make_tmap_sw128(&tmA, codebook, (uint64_t)shape->Hkv * shape->L, kD, 128));
  if (rc) return rc;
  tmC = tmA;
  if (append) {
    EncArgs e;
    e.keys = static_cast<const uint16_t*>(k_cache);
    e.chat = static_cast<const uint16_t*>(chat);
    e.nrm = nrm;
    e.slot = reinterpret_cast<unsigned long long*>(base + Lw.eslot);
    e.counter = reinterpret_cast<unsigned int*>(base + Lw.ectr);
    e.codes = shape->code_bytes == 1 ? nullptr : codes;
    e.codes8 = shape->code_bytes == 1 ? reinterpret_cast<uint8_t*>(codes) : nullptr;
    e.hist = nullptr;  // the select kernel adds it
    e.B = shape->B;
    e.Hkv = shape->Hkv;
    e.L = shape->L;
    e.n_max = shape->n_max;
    e.t_begin = n_ctx - 1;
    e.T = 1;
    e.nvec = shape->B;
    e.lsplit = e.tiles_per_split = 0;
    prep_set_encode(p, e);
    rc = cuda_status(make_tmap_sw128(&tmC, chat, (uint64_t)shape->Hkv * shape->L, 2 * kD, encode_codeword_tile()));
    if (rc) return rc;
  }
  prep_balance(p);
  stage_mark(0, st);
  if (la.qt) {
    rc = cuda_status(launch_qprep(la, st));
    if (rc) return rc;
  }
  if (lut_fma) {
    rc = cuda_status(launch_lut_fma(la, st));
    if (rc) return rc;
  }
  if (lut_persist) {
    rc = cuda_status(launch_lut_persist(la, tmA, st));
    if (rc) return rc;
  }
  rc = cuda_status(launch_prep(p, tmA, tmC, st));
  if (rc) return rc;
  stage_mark(1, st);

  // a3 + a4
  if (d.keff > 0 || (append && hist)) {
    SelArgs sa{};
    sa.agg = agg;
    sa.hist = hist;
    sa.append = append ? 1 : 0;
    sa.append_hist = append ? 1 : 0;
    sa.hist_end = n_ctx - (append ? 1 : 0) - params->hist_lag;  // hist covers [0, hist_end)
    sa.codes = codes;
    sa.codes8 = shape->code_bytes == 1 ? reinterpret_cast<const uint8_t*>(codes) : nullptr;
    sa.sel = sel;
    sa.pinfo = reinterpret_cast<uint32_t*>(base + Lw.pinfo);
    sa.tblg = reinterpret_cast<uint32_t*>(base + Lw.tblg);
    sa.desc = reinterpret_cast<unsigned long long*>(base + Lw.desc);
    sa.tickets = reinterpret_cast<unsigned int*>(base + Lw.tick);
    sa.desc_stride = shape->n_max / select_chunk_tokens() + 2;
    sa.nchunk = nchunk;
    sa.B = shape->B;
    sa.wlog = nullptr;
    sa.P = d.P;
    if ((long_select || post_select) && attend && n_wl > 0) {  // the threshold kernel computes the window logits before its wait
      sa.wlog = wlog;
      sa.q = static_cast<const uint16_t*>(q);
      sa.kc = static_cast<const uint16_t*>(k_cache);
      sa.Hq = shape->Hq;
      sa.G = d.G;
      sa.n_wl = n_wl;
      sa.win_lo = d.w0;
      sa.scale_log2 = kScaleLog2;
      sa.rt = la.rt;
    }
    sa.L = shape->L;
    sa.W = d.W;
    sa.n_max = shape->n_max;
    sa.n_ctx = n_ctx;
    sa.c0 = d.c0;
    sa.c1 = d.c1;
    sa.n_s = d.n_s;
    sa.w0 = d.w0;
    sa.keff = d.keff;
    sa.sel_stride = std::max(d.keff, 1);
    sa.shard_begin = 0;
    sa.shard_len = shape->n_max;
    sa.rank = 0;
    // one CTA per pair while the candidates fit one code chunk; beyond, one streaming CTA per
    // pair (hist given) or threshold + chunked scan (counts need a pass over the codes)
    CUtensorMap tmK;
    if (pipe_select) {
      rc = cuda_status(make_tmap_codes(&tmK, codes, (uint64_t)d.P, (uint64_t)shape->n_max));
      if (rc) return rc;
    }
    if (post_select) {
      const PostingsLayout pl = postings_layout(shape);
      sa.post_off = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(postings) + pl.off);
      sa.post_tok = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(postings) + pl.tok);
      sa.n_post = n_post;
      sa.pbits = reinterpret_cast<uint32_t*>(base + Lw.pbits);
      sa.pbits_stride = postings_bits_stride(shape->n_max);
    }
    rc = cuda_status(post_select    ? launch_select_postings(sa, st)
                     : pipe_select  ? launch_select_pipe(sa, tmK, std::min(sm_count(), 2 * d.P), st)
                     : split_select ? launch_select_split(sa, d.P, st)
                                    : launch_select(sa, d.P, st));
    if (rc) return rc;
  }
  stage_mark(2, st);
  if (!attend) return A2ATS_OK;

  // a5 + a6
  AttnArgs aa;
  aa.q = static_cast<const uint16_t*>(q);
  std::memcpy(aa.bcs, la.bcs, sizeof(aa.bcs));
  aa.wlog = wlog;
  aa.wlog_late = (long_select || post_select) ? 1 : 0;  // (the select kernel wrote wlog)
  aa.win_as_bridge = rope_std ? 1 : 0;
  aa.n_wl = n_wl;
  aa.cs = cs;
  aa.kc = static_cast<const uint16_t*>(k_cache);
  aa.vc = static_cast<const uint16_t*>(v_cache);
  aa.sel = sel;
  aa.part = reinterpret_cast<float*>(base + Lw.part);
  aa.counter = reinterpret_cast<unsigned int*>(base + Lw.actr);
  aa.out = out;
  aa.nsel = nullptr;
  aa.part_out = nullptr;
  aa.Hq = shape->Hq;
  aa.Hkv = shape->Hkv;
  aa.G = d.G;
  aa.n_max = shape->n_max;
  aa.n_ctx = n_ctx;
  aa.keff = d.keff;
  aa.sel_stride = d.keff;
  aa.R = d.R;
  aa.nsplit = d.nsplit;
  aa.n_s = d.n_s;
  aa.sink_lo = 0;
  aa.n_w = d.n_w;
  aa.win_lo = d.w0;
  aa.shard_begin = 0;
  aa.scale_log2 = kScaleLog2;
  rc = cuda_status(launch_attention(aa, d.P, d.GT, st));
  if (rc) return rc;
  stage_mark(3, st);

  if (scores_out) {
    rc = cuda_status(launch_scores(lut_full, codes, scores_out, shape->B, shape->Hq, shape->Hkv, d.G, shape->L,
                                   shape->n_max, n_ctx, st));
    if (rc) return rc;
  }
  stage_mark(4, st);
  return A2ATS_OK;
}
}  // namespace

extern "C" {

int a2ats_decode_step(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                      const void* k_cache, const void* v_cache, const uint16_t* codes, const void* codebook,
                      const int32_t* hist, float* out, int32_t* sel_out, float* scores_out, void* ws,
                      size_t ws_bytes, void* stream) {
  return decode_impl(shape, params, n_ctx, q, k_cache, v_cache, const_cast<uint16_t*>(codes), codebook,
                     const_cast<int32_t*>(hist), nullptr, nullptr, out, sel_out, scores_out, ws, ws_bytes, stream);
}

int a2ats_decode_step_append(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                             const void* k_cache, const void* v_cache, uint16_t* codes, const void* codebook,
                             int32_t* hist, const void* chat, const float* nrm, float* out, int32_t* sel_out,
                             float* scores_out, void* ws, size_t ws_bytes, void* stream) {
  if (!chat) return A2ATS_EINVAL;
  return decode_impl(shape, params, n_ctx, q, k_cache, v_cache, codes, codebook, hist, chat, nrm, out, sel_out,
                     scores_out, ws, ws_bytes, stream);
}

int a2ats_select_topk(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                      const uint16_t* codes, const void* codebook, const int32_t* hist, int32_t* sel_out, void* ws,
                      size_t ws_bytes, void* stream) {
  return decode_impl(shape, params, n_ctx, q, nullptr, nullptr, const_cast<uint16_t*>(codes), codebook,
                     const_cast<int32_t*>(hist), nullptr, nullptr, nullptr, sel_out, nullptr, ws, ws_bytes, stream,
                     false);
}

// ------------------------------------------------------------------ posting-list selection (f3)
size_t a2ats_postings_bytes(const a2ats_shape* shape) {
  if (check_shape(shape)) return 0;
  return postings_layout(shape).total;
}

int a2ats_postings_build(const a2ats_shape* shape, const uint16_t* codes, int32_t n_tokens, void* postings,
                         void* stream) {
  int rc = check_shape(shape);
  if (rc) return rc;
  if (!codes || !postings || n_tokens < 0 || n_tokens > shape->n_max || !aligned16(postings)) return A2ATS_EINVAL;
  const PostingsLayout pl = postings_layout(shape);
  uint8_t* b = static_cast<uint8_t*>(postings);
  return cuda_status(launch_postings_build(codes, shape->code_bytes == 1, shape->B * shape->Hkv, shape->n_max,
                                           shape->L, n_tokens,
                                           reinterpret_cast<int32_t*>(b + pl.off),
                                           reinterpret_cast<int32_t*>(b + pl.tok), static_cast<cudaStream_t>(stream)));
}

int a2ats_select_topk_postings(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                               const uint16_t* codes, const void* codebook, const int32_t* hist,
                               const void* postings, int32_t n_post, int32_t* sel_out, void* ws, size_t ws_bytes,
                               void* stream) {
  if (!postings || !hist || n_post < 0 || n_post > n_ctx) return A2ATS_EINVAL;
  if (check_shape(shape)) return A2ATS_EINVAL;
  if (!select_postings_ok(shape->L, n_ctx)) return A2ATS_EUNSUPPORTED;
  return decode_impl(shape, params, n_ctx, q, nullptr, nullptr, const_cast<uint16_t*>(codes), codebook,
                     const_cast<int32_t*>(hist), nullptr, nullptr, nullptr, sel_out, nullptr, ws, ws_bytes, stream,
                     false, postings, n_post);
}

int a2ats_decode_step_postings(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, const void* q,
                               const void* k_cache, const void* v_cache, const uint16_t* codes,
                               const void* codebook, const int32_t* hist, const void* postings, int32_t n_post,
                               float* out, int32_t* sel_out, void* ws, size_t ws_bytes, void* stream) {
  if (!postings || !hist || n_post < 0 || n_post > n_ctx) return A2ATS_EINVAL;
  if (check_shape(shape)) return A2ATS_EINVAL;
  if (!select_postings_ok(shape->L, n_ctx)) return A2ATS_EUNSUPPORTED;
  return decode_impl(shape, params, n_ctx, q, k_cache, v_cache, const_cast<uint16_t*>(codes), codebook,
                     const_cast<int32_t*>(hist), nullptr, nullptr, out, sel_out, nullptr, ws, ws_bytes, stream, true,
                     postings, n_post);
}

int a2ats_decode_step_append_postings(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx,
                                      const void* q, const void* k_cache, const void* v_cache, uint16_t* codes,
                                      const void* codebook, int32_t* hist, const void* chat, const float* nrm,
                                      const void* postings, int32_t n_post, float* out, int32_t* sel_out, void* ws,
                                      size_t ws_bytes, void* stream) {
  if (!chat || !postings || !hist || n_post < 0 || n_post > n_ctx - 1) return A2ATS_EINVAL;
  if (check_shape(shape)) return A2ATS_EINVAL;
  if (!select_postings_ok(shape->L, n_ctx)) return A2ATS_EUNSUPPORTED;
  return decode_impl(shape, params, n_ctx, q, k_cache, v_cache, codes, codebook, hist, chat, nrm, out, sel_out,
                     nullptr, ws, ws_bytes, stream, true, postings, n_post);
}

// ------------------------------------------------------------------ end-to-end staging
namespace a2ats {
// one 16-B piece per thread: q pieces first, then the key rows, then the value rows
__global__ __launch_bounds__(256) void stage_rows_kernel(const uint4* q_src, const uint4* k_src, const uint4* v_src,
                                                         uint4* q_dst, uint8_t* k_cache, uint8_t* v_cache, int nq,
                                                         int nkv, int n_max, int row) {
  pdl_wait();  // the previous step reads q and the caches
  // no early pdl_trigger(): the next kernel's pre-wait prologue reads q and the new K/V rows
  // written here, so dependents launch only at this grid's completion (implicit trigger)
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    if (q_src) q_dst[i] = q_src[i];
    return;
  }
  i -= nq;
  const bool val = i >= nkv;
  if (val) i -= nkv;
  if (i >= nkv) return;
  const uint4* src = val ? v_src : k_src;
  if (!src) return;
  const int pair = i >> 4, c = i & 15;  // 16 pieces of 16 B per 256-B row
  uint8_t* dst = (val ? v_cache : k_cache) + ((size_t)pair * n_max + row) * 256 + c * 16;
  *reinterpret_cast<uint4*>(dst) = src[i];
}
}  // namespace a2ats

extern "C" int a2ats_stage_rows(const a2ats_shape* shape, int32_t n_ctx, const void* q_src, const void* k_src,
                                const void* v_src, void* q_dst, void* k_cache, void* v_cache, void* stream) {
  int rc = check_shape(shape);
  if (rc) return rc;
  if (n_ctx <= 0 || n_ctx > shape->n_max) return A2ATS_EINVAL;
  if ((q_src && (!q_dst || !aligned16(q_src) || !aligned16(q_dst))) ||
      (k_src && (!k_cache || !aligned16(k_src) || !aligned16(k_cache))) ||
      (v_src && (!v_cache || !aligned16(v_src) || !aligned16(v_cache))))
    return A2ATS_EINVAL;
  const int nq = shape->B * shape->Hq * (kD / 8), nkv = shape->B * shape->Hkv * (kD / 8);
  const int n = nq + 2 * nkv;
  return cuda_status(launch_pdl(a2ats::stage_rows_kernel, dim3((n + 255) / 256), dim3(256), 0,
                                static_cast<cudaStream_t>(stream), static_cast<const uint4*>(q_src),
                                static_cast<const uint4*>(k_src), static_cast<const uint4*>(v_src),
                                static_cast<uint4*>(q_dst), static_cast<uint8_t*>(k_cache),
                                static_cast<uint8_t*>(v_cache), nq, nkv, shape->n_max, n_ctx - 1));
}

}  // extern "C"

// ------------------------------------------------------------------ sequence-sharded step
// SURVEY 8b / 8e / 8f.1 (the paper itself is single-GPU).  Rank r holds the global
// tokens [bounds[r], bounds[r + 1]) of every (b, KV head) sequence in its own K / V / code
// arrays (local index = global - bounds[r]); q, the codebook and the shard STATE are
// replicated.  One step = a0 for the new token n-1 on its owner + the LUT (bitwise identical on
// every rank) + the collective-free global top-K from the replicated histograms + the local
// attention partial, then ONE all-gather (every rank's partial (m, l, o) and the new token's
// code) and the finish: LSE combine in rank order + the state update (the new code joins the
// replicated histograms, the code ring and, for the first tokens, the sink codes).
namespace a2ats {
namespace {

// NCCL through dlopen (the process's libnccl.so.2: the one torch.distributed loaded, or the
// path in A2ATS_NCCL_LIB): no link-time dependency, a build without NCCL still loads.
struct NcclApi {
  bool ok = false;
  int (*get_unique_id)(void*) = nullptr;
  int (*comm_init_rank)(void**, int, a2ats_comm_id, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
};
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi x;
    const char* path = std::getenv("A2ATS_NCCL_LIB");
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
    if (!h) h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
    x.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
    x.comm_init_rank = reinterpret_cast<int (*)(void**, int, a2ats_comm_id, int)>(dlsym(h, "ncclCommInitRank"));
    x.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
    x.all_gather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
        dlsym(h, "ncclAllGather"));
    x.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(h, "ncclAllReduce"));
    x.ok = x.get_unique_id && x.comm_init_rank && x.comm_destroy && x.all_gather && x.all_reduce;
    return x;
  }();
  return api;
}
constexpr int kNcclInt32 = 2, kNcclFloat32 = 7, kNcclSum = 0;  // ncclDataType_t / ncclRedOp_t values

struct ShardState {  // offsets in the caller's state buffer (a2ats_shard_state_bytes)
  size_t hist_g, hist_r, ring, sinkc, total;
  int WR, n_sink_cap;
};
ShardState state_layout(const a2ats_shape* s, const a2ats_params* p, int world) {
  ShardState st;
  const size_t P = (size_t)s->B * s->Hkv;
  st.WR = 1;
  while (st.WR < p->window) st.WR <<= 1;
  st.n_sink_cap = std::max(p->n_sink, 1);
  size_t o = 0;
  st.hist_g = o; o = align_up(o + P * s->L * 4);
  st.hist_r = o; o = align_up(o + (size_t)world * P * s->L * 4);
  st.ring = o; o = align_up(o + P * st.WR * 2);
  st.sinkc = o; o = align_up(o + P * st.n_sink_cap * 2);
  st.total = o;
  return st;
}
size_t msg_floats(const a2ats_shape* s) {  // partial [B*Hq][130] + the new token's code per pair
  return ((size_t)s->B * s->Hq * 130 + (size_t)s->B * s->Hkv + 3) / 4 * 4;
}
struct ShardWs {
  size_t dec, msg, recv, nsel, total;
};
ShardWs shard_ws_layout(const a2ats_shape* s, const a2ats_params* p, int world) {
  ShardWs w;
  size_t o = 0;
  w.dec = o; o = align_up(o + decode_layout(s, p).total);
  w.msg = o; o = align_up(o + msg_floats(s) * 4);
  w.recv = o; o = align_up(o + (size_t)world * msg_floats(s) * 4);
  w.nsel = o; o = align_up(o + (size_t)s->B * s->Hkv * 4);
  w.total = o;
  return w;
}

int check_bounds(const int32_t* bounds, int world, int rank, const a2ats_shape* s) {
  if (!bounds || world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return A2ATS_EINVAL;
  if (bounds[0] != 0) return A2ATS_EINVAL;
  for (int r = 0; r < world; ++r)
    if (bounds[r + 1] < bounds[r]) return A2ATS_EINVAL;
  if (bounds[rank + 1] - bounds[rank] > s->n_max) return A2ATS_EINVAL;
  return A2ATS_OK;
}
int owner_of_host(const int32_t* bounds, int world, int t) {
  for (int r = 0; r < world; ++r)
    if (t >= bounds[r] && t < bounds[r + 1]) return r;
  return -1;
}

// state of tokens [0, n): local histogram (hist_r[rank], hist_g) and the codes of the sinks and
// the latest WR tokens held by this rank; other entries 0 (summed across ranks by the caller)
__global__ void shard_state_local_kernel(const uint16_t* codes, int n_max, int L, int P, int lo, int hi, int n,
                                         int rank, int WR, int n_sink_cap, int32_t* hist_g, int32_t* hist_r,
                                         int32_t* ring32, int32_t* sink32) {
  const int pair = blockIdx.y;
  const uint16_t* cp = codes + (size_t)pair * n_max;
  const int e = min(hi, n);
  for (int t = lo + blockIdx.x * blockDim.x + threadIdx.x; t < e; t += gridDim.x * blockDim.x) {
    const int code = cp[t - lo];
    atomicAdd(&hist_g[(size_t)pair * L + code], 1);
    atomicAdd(&hist_r[((size_t)rank * P + pair) * L + code], 1);
    if (t >= n - WR) ring32[(size_t)pair * WR + (t % WR)] = code;
    if (t < n_sink_cap) sink32[(size_t)pair * n_sink_cap + t] = code;
  }
}
__global__ void shard_state_pack_kernel(const int32_t* ring32, const int32_t* sink32, uint16_t* ring,
                                        uint16_t* sinkc, int nring, int nsink) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nring + nsink; i += gridDim.x * blockDim.x) {
    if (i < nring) ring[i] = (uint16_t)ring32[i];
    else sinkc[i - nring] = (uint16_t)sink32[i - nring];
  }
}
// finish: the new token's code (from its owner's message) joins the replicated state
__global__ void shard_state_update_kernel(const float* msgs, size_t msg_stride, size_t code_off, int owner, int P,
                                          int L, int t_new, int WR, int n_sink_cap, int32_t* hist_g,
                                          int32_t* hist_r, uint16_t* ring, uint16_t* sinkc) {
  pdl_wait();
  pdl_trigger();
  const int pair = blockIdx.x * blockDim.x + threadIdx.x;
  if (pair >= P) return;
  const uint32_t code = reinterpret_cast<const uint32_t*>(msgs + (size_t)owner * msg_stride + code_off)[pair];
  if (code >= (uint32_t)L) return;  // (never: the encoder emits codes < L)
  hist_g[(size_t)pair * L + code] += 1;
  hist_r[((size_t)owner * P + pair) * L + code] += 1;
  ring[(size_t)pair * WR + (t_new % WR)] = (uint16_t)code;
  if (t_new < n_sink_cap) sinkc[(size_t)pair * n_sink_cap + t_new] = (uint16_t)code;
}

}  // namespace
}  // namespace a2ats

extern "C" {

int a2ats_comm_unique_id(void* id) {
  if (!id) return A2ATS_EINVAL;
  if (!nccl().ok) return A2ATS_ENCCL;
  return nccl().get_unique_id(id) == 0 ? A2ATS_OK : A2ATS_ENCCL;
}

struct a2ats_comm {
  void* nccl_comm;
  int world, rank;
};

int a2ats_comm_init(const void* id, int32_t world, int32_t rank, a2ats_comm** out) {
  if (!id || !out || world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return A2ATS_EINVAL;
  if (!nccl().ok) return A2ATS_ENCCL;
  a2ats_comm_id uid;
  std::memcpy(&uid, id, sizeof(uid));
  void* c = nullptr;
  if (nccl().comm_init_rank(&c, world, uid, rank) != 0) return A2ATS_ENCCL;
  *out = new a2ats_comm{c, world, rank};
  return A2ATS_OK;
}

int a2ats_comm_destroy(a2ats_comm* comm) {
  if (!comm) return A2ATS_EINVAL;
  const int r = nccl().ok && nccl().comm_destroy(comm->nccl_comm) == 0 ? A2ATS_OK : A2ATS_ENCCL;
  delete comm;
  return r;
}

size_t a2ats_shard_state_bytes(const a2ats_shape* shape, const a2ats_params* params, int32_t world) {
  if (check_shape(shape) || check_params(params) || world < 1 || world > kMaxRanks) return 0;
  return state_layout(shape, params, world).total;
}
int a2ats_shard_state_layout(const a2ats_shape* shape, const a2ats_params* params, int32_t world, size_t* offsets) {
  if (check_shape(shape) || check_params(params) || world < 1 || world > kMaxRanks || !offsets) return A2ATS_EINVAL;
  const ShardState st = state_layout(shape, params, world);
  offsets[0] = st.hist_g;
  offsets[1] = st.hist_r;
  offsets[2] = st.ring;
  offsets[3] = st.sinkc;
  offsets[4] = (size_t)st.WR;
  offsets[5] = (size_t)st.n_sink_cap;
  return A2ATS_OK;
}
size_t a2ats_shard_msg_bytes(const a2ats_shape* shape) {
  if (check_shape(shape)) return 0;
  return msg_floats(shape) * 4;
}
size_t a2ats_shard_workspace_bytes(const a2ats_shape* shape, const a2ats_params* params, int32_t world) {
  if (check_shape(shape) || check_params(params) || world < 1 || world > kMaxRanks) return 0;
  return shard_ws_layout(shape, params, world).total;
}

int a2ats_shard_state_build(const a2ats_shape* shape, const a2ats_params* params, int32_t world, int32_t rank,
                            const int32_t* bounds, int32_t n_tokens, const uint16_t* codes, void* state, void* ws,
                            size_t ws_bytes, a2ats_comm* comm, void* stream) {
  int rc = check_shape(shape);
  if (!rc) rc = check_params(params);
  if (!rc) rc = check_bounds(bounds, world, rank, shape);
  if (rc) return rc;
  if (shape->code_bytes == 1) return A2ATS_EUNSUPPORTED;
  if (!codes || !state || n_tokens < 0 || n_tokens > bounds[world]) return A2ATS_EINVAL;
  if (comm && (comm->world != world || comm->rank != rank)) return A2ATS_EINVAL;
  const ShardWs W = shard_ws_layout(shape, params, world);
  const ShardState S = state_layout(shape, params, world);
  const int P = shape->B * shape->Hkv;
  const size_t nring = (size_t)P * S.WR, nsink = (size_t)P * S.n_sink_cap;
  if (!ws || ws_bytes < W.total || (size_t)world * msg_floats(shape) * 4 < (nring + nsink) * 4) return A2ATS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* sb = static_cast<uint8_t*>(state);
  // scratch: the message receive area (the step's zero-on-entry counters must stay untouched)
  int32_t* ring32 = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + W.recv);
  int32_t* sink32 = ring32 + nring;
  rc = cuda_status(cudaMemsetAsync(state, 0, S.total, st));
  if (!rc) rc = cuda_status(cudaMemsetAsync(ws, 0, (nring + nsink) * 4, st));
  if (rc) return rc;
  dim3 grid(std::max(1, std::min(64, (bounds[rank + 1] - bounds[rank] + 1023) / 1024)), P);
  shard_state_local_kernel<<<grid, 256, 0, st>>>(codes, shape->n_max, shape->L, P, bounds[rank], bounds[rank + 1],
                                                  n_tokens, rank, S.WR, S.n_sink_cap,
                                                  reinterpret_cast<int32_t*>(sb + S.hist_g),
                                                  reinterpret_cast<int32_t*>(sb + S.hist_r), ring32, sink32);
  rc = cuda_status(cudaGetLastError());
  if (rc) return rc;
  if (world > 1 && comm) {  // every rank's entries are zero elsewhere: sums assemble the replicated state
    const size_t nh = (size_t)(world + 1) * P * shape->L;  // hist_g and hist_r are adjacent int32 arrays
    if (S.hist_r != S.hist_g + align_up((size_t)P * shape->L * 4)) return A2ATS_EINVAL;
    int r1 = nccl().all_reduce(sb + S.hist_g, sb + S.hist_g, (size_t)P * shape->L, kNcclInt32, kNcclSum,
                               comm->nccl_comm, st);
    int r2 = nccl().all_reduce(sb + S.hist_r, sb + S.hist_r, (size_t)world * P * shape->L, kNcclInt32, kNcclSum,
                               comm->nccl_comm, st);
    int r3 = nccl().all_reduce(ring32, ring32, nring + nsink, kNcclInt32, kNcclSum, comm->nccl_comm, st);
    (void)nh;
    if (r1 || r2 || r3) return A2ATS_ENCCL;
  }
  shard_state_pack_kernel<<<64, 256, 0, st>>>(ring32, sink32, reinterpret_cast<uint16_t*>(sb + S.ring),
                                             reinterpret_cast<uint16_t*>(sb + S.sinkc), (int)nring, (int)nsink);
  return cuda_status(cudaGetLastError());
}

}  // extern "C"

namespace a2ats {
namespace {
int shard_common(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world, int32_t rank,
                 const int32_t* bounds) {
  int rc = check_shape(shape);
  if (!rc) rc = check_params(params);
  if (!rc) rc = check_bounds(bounds, world, rank, shape);
  if (rc) return rc;
  if (n_ctx <= 0 || n_ctx > bounds[world]) return A2ATS_EINVAL;
  if (owner_of_host(bounds, world, n_ctx - 1) < 0) return A2ATS_EINVAL;
  if (params->kv_location != A2ATS_KV_DEVICE || shape->code_bytes == 1 || params->hist_lag ||
      params->rope_mode != A2ATS_ROPE_WINDOWED)
    return A2ATS_EUNSUPPORTED;
  if (shape->n_max % 64 || !select_pipe_ok(shape->L) || shape->B > encode_cw_max()) return A2ATS_EUNSUPPORTED;
  return A2ATS_OK;
}

// phase A: a0 (owner) + LUT + global threshold from the state + local scan + local attention
// partial, into this rank's message [msg_floats]
int shard_partial(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world, int32_t rank,
                  const int32_t* bounds, const void* q, const void* k_cache, const void* v_cache, uint16_t* codes,
                  const void* codebook, const void* chat, const float* nrm, const void* state, float* msg,
                  int32_t* sel_out, void* ws, size_t ws_bytes, cudaStream_t st, float* out_direct = nullptr) {
  int rc = shard_common(shape, params, n_ctx, world, rank, bounds);
  if (rc) return rc;
  if (!q || !k_cache || !v_cache || !codes || !codebook || !chat || !nrm || !state || !msg) return A2ATS_EINVAL;
  if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(codes) || !aligned16(codebook) ||
      !aligned16(chat) || !aligned16(msg))
    return A2ATS_EINVAL;
  const ShardWs W = shard_ws_layout(shape, params, world);
  if (!ws || ws_bytes < W.total) return A2ATS_EWORKSPACE;
  const DecodeWs Lw = decode_layout(shape, params);
  const ShardState S = state_layout(shape, params, world);
  Derived d;
  derive(shape, params, n_ctx, &d);
  uint8_t* base = static_cast<uint8_t*>(ws) + W.dec;
  const uint8_t* sb = static_cast<const uint8_t*>(state);
  const int lo = bounds[rank], hi = bounds[rank + 1];
  const int owner = owner_of_host(bounds, world, n_ctx - 1);
  const int kcap = std::max(1, (int)std::min<long long>(params->topk, shape->n_max));
  int32_t* sel = sel_out ? sel_out : reinterpret_cast<int32_t*>(base + Lw.sel);
  int32_t* nsel = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + W.nsel);
  float* wlog = reinterpret_cast<float*>(base + Lw.wlog);
  float* agg = reinterpret_cast<float*>(base + Lw.agg);

  // 1. prep: LUT (every rank: bitwise identical), the new token's code (owner), the logits of
  //    this rank's window rows
  LutArgs la = make_lut_args(shape, params, d, q, codebook, agg, nullptr, reinterpret_cast<float2*>(base + Lw.cs));
  const bool lut_fma = params->lut_engine == A2ATS_LUT_FMA ||
                       (params->lut_engine == A2ATS_LUT_AUTO && shape->B * d.G <= A2ATS_LUT_FMA_MAX_VECTORS);
  if (la.NV > A2ATS_QPREP_MIN_NV && !lut_fma) la.qt = reinterpret_cast<uint16_t*>(base + Lw.qt);
  PrepArgs p = prep_empty();
  prep_set_lut(p, la);
  if (lut_fma) p.n_lut = 0;
  const int w_lo = std::max(d.w0, lo), w_hi = std::min(n_ctx, hi);
  prep_set_window(p, shape, k_cache, wlog, n_ctx, w_lo, std::max(0, w_hi - w_lo), lo);
  const int n_wl = p.n_wl;
  p.n_win = 0;  // the window-row logits are computed by the threshold kernel before its wait
  CUtensorMap tmA, tmC;
  rc = cuda_status(make_tmap_sw128(&tmA, codebook, (uint64_t)shape->Hkv * shape->L, kD, 128));
  if (rc) return rc;
  tmC = tmA;
  if (rank == owner) {
    EncArgs e;
    e.keys = static_cast<const uint16_t*>(k_cache);
    e.chat = static_cast<const uint16_t*>(chat);
    e.nrm = nrm;
    e.slot = reinterpret_cast<unsigned long long*>(base + Lw.eslot);
    e.counter = reinterpret_cast<unsigned int*>(base + Lw.ectr);
    e.codes = codes;
    e.hist = nullptr;  // the state update (finish) adds the new code everywhere
    e.B = shape->B;
    e.Hkv = shape->Hkv;
    e.L = shape->L;
    e.n_max = shape->n_max;
    e.t_begin = n_ctx - 1 - lo;
    e.T = 1;
    e.nvec = shape->B;
    e.lsplit = e.tiles_per_split = 0;
    prep_set_encode(p, e);
    rc = cuda_status(make_tmap_sw128(&tmC, chat, (uint64_t)shape->Hkv * shape->L, 2 * kD, encode_codeword_tile()));
    if (rc) return rc;
  }
  prep_balance(p);
  stage_mark(0, st);
  if (la.qt) {
    rc = cuda_status(launch_qprep(la, st));
    if (rc) return rc;
  }
  if (lut_fma) {
    rc = cuda_status(launch_lut_fma(la, st));
    if (rc) return rc;
  }
  rc = cuda_status(launch_prep(p, tmA, tmC, st));
  if (rc) return rc;
  stage_mark(1, st);

  // 2. global threshold from the replicated state + this rank's tie share; local scan
  SelArgs sa{};
  sa.agg = agg;
  sa.codes = codes;
  sa.sel = sel;
  sa.sel_stride = kcap;
  sa.L = shape->L;
  sa.W = d.W;
  sa.n_max = shape->n_max;
  sa.n_ctx = n_ctx;
  sa.hist_end = n_ctx;  // (the shard kernels count from the replicated state, not load_cnt)
  sa.n_s = d.n_s;
  sa.w0 = d.w0;
  sa.keff = d.keff;  // global K_eff
  sa.P = d.P;
  sa.B = shape->B;
  sa.shard_begin = lo;
  sa.shard_len = hi - lo;
  sa.rank = rank;
  sa.world = world;
  sa.owner = owner;
  for (int r = 0; r <= world; ++r) sa.bounds[r] = bounds[r];
  sa.hist_g = reinterpret_cast<const int32_t*>(sb + S.hist_g);
  sa.hist_r = reinterpret_cast<const int32_t*>(sb + S.hist_r);
  sa.ring = reinterpret_cast<const uint16_t*>(sb + S.ring);
  sa.sinkc = reinterpret_cast<const uint16_t*>(sb + S.sinkc);
  sa.WR = S.WR;
  sa.n_sink_cap = S.n_sink_cap;
  sa.send_codes = reinterpret_cast<uint32_t*>(msg + (size_t)shape->B * shape->Hq * 130);
  sa.pinfo = reinterpret_cast<uint32_t*>(base + Lw.pinfo);
  sa.tblg = reinterpret_cast<uint32_t*>(base + Lw.tblg);
  sa.nsel_out = nsel;
  // the scan's range: this rank's part of the candidates [c0, c1), in local indices
  const int lc0 = std::max(d.c0, lo), lc1 = std::min(d.c1, hi);
  sa.c0 = lc1 > lc0 ? lc0 - lo : 0;
  sa.c1 = lc1 > lc0 ? lc1 - lo : 0;
  sa.sel_base = lo;
  if (n_wl > 0) {  // this rank's window rows: logits in the threshold kernel's prologue
    sa.wlog = wlog;
    sa.q = static_cast<const uint16_t*>(q);
    sa.kc = static_cast<const uint16_t*>(k_cache);
    sa.Hq = shape->Hq;
    sa.G = d.G;
    sa.n_wl = n_wl;
    sa.win_lo = w_lo;
    sa.scale_log2 = kScaleLog2;
    sa.rt = la.rt;
  }
  const int nblk = (lc1 > lc0 && d.keff > 0) ? std::min(sm_count(), 2 * d.P) : 0;
  CUtensorMap tmK;
  rc = cuda_status(make_tmap_codes(&tmK, codes, (uint64_t)d.P, (uint64_t)shape->n_max));
  if (rc) return rc;
  rc = cuda_status(launch_select_shard(sa, tmK, nblk, st));
  if (rc) return rc;
  stage_mark(2, st);

  // 3. attention over this rank's rows of Sel -> partial (m, l, o) into the message
  const int s_lo = std::max(0, lo), s_hi = std::min(d.n_s, hi);
  AttnArgs aa;
  aa.q = static_cast<const uint16_t*>(q);
  std::memcpy(aa.bcs, la.bcs, sizeof(aa.bcs));
  aa.wlog = wlog;
  aa.wlog_late = 1;  // (the shard threshold kernel writes wlog)
  aa.win_as_bridge = 0;
  aa.n_wl = n_wl;
  aa.cs = reinterpret_cast<float2*>(base + Lw.cs);
  aa.kc = static_cast<const uint16_t*>(k_cache);
  aa.vc = static_cast<const uint16_t*>(v_cache);
  aa.sel = sel;
  aa.nsel = nsel;
  aa.part = reinterpret_cast<float*>(base + Lw.part);
  aa.counter = reinterpret_cast<unsigned int*>(base + Lw.actr);
  aa.out = out_direct;  // one rank: the normalised output directly (no combine)
  aa.part_out = out_direct ? nullptr : msg;
  aa.Hq = shape->Hq;
  aa.Hkv = shape->Hkv;
  aa.G = d.G;
  aa.n_max = shape->n_max;
  aa.n_ctx = n_ctx;
  aa.keff = d.keff;
  aa.sel_stride = kcap;
  aa.R = d.R;
  aa.n_s = std::max(0, s_hi - s_lo);
  aa.sink_lo = s_lo;
  aa.n_w = std::max(0, w_hi - w_lo);
  aa.win_lo = w_lo;
  aa.shard_begin = lo;
  const int local_cand = std::max(0, lc1 - lc0);
  const int mmax = aa.n_s + std::min(d.keff, local_cand) + aa.n_w;
  aa.nsplit = std::max(1, (mmax + d.R - 1) / d.R);
  aa.scale_log2 = kScaleLog2;
  rc = cuda_status(launch_attention(aa, d.P, d.GT, st));
  if (rc) return rc;
  stage_mark(3, st);
  return A2ATS_OK;
}

// phase B: LSE combine of the world's partials in rank order + the state update
int shard_finish(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world,
                 const int32_t* bounds, const float* msgs, void* state, float* out, cudaStream_t st,
                 bool combine = true) {
  const ShardState S = state_layout(shape, params, world);
  const int owner = owner_of_host(bounds, world, n_ctx - 1);
  const size_t mf = msg_floats(shape);
  const int P = shape->B * shape->Hkv;
  int rc = A2ATS_OK;
  if (combine) rc = cuda_status(launch_combine(msgs, world, shape->B * shape->Hq, mf, out, st));
  if (rc) return rc;
  uint8_t* sb = static_cast<uint8_t*>(state);
  rc = cuda_status(launch_pdl(shard_state_update_kernel, dim3((P + 255) / 256), dim3(256), 0, st, msgs, mf,
                              (size_t)shape->B * shape->Hq * 130, owner, P, shape->L, n_ctx - 1, S.WR,
                              S.n_sink_cap, reinterpret_cast<int32_t*>(sb + S.hist_g),
                              reinterpret_cast<int32_t*>(sb + S.hist_r), reinterpret_cast<uint16_t*>(sb + S.ring),
                              reinterpret_cast<uint16_t*>(sb + S.sinkc)));
  stage_mark(4, st);
  return rc;
}
}  // namespace
}  // namespace a2ats

extern "C" {

int a2ats_shard_step_partial(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world,
                             int32_t rank, const int32_t* bounds, const void* q, const void* k_cache,
                             const void* v_cache, uint16_t* codes, const void* codebook, const void* chat,
                             const float* nrm, const void* state, void* msg, int32_t* sel_out, void* ws,
                             size_t ws_bytes, void* stream) {
  return shard_partial(shape, params, n_ctx, world, rank, bounds, q, k_cache, v_cache, codes, codebook, chat, nrm,
                       state, static_cast<float*>(msg), sel_out, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int a2ats_shard_step_finish(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world,
                            const int32_t* bounds, const void* msgs, void* state, float* out, void* stream) {
  int rc = shard_common(shape, params, n_ctx, world, 0, bounds);
  if (rc) return rc;
  if (!msgs || !state || !out || !aligned16(msgs)) return A2ATS_EINVAL;
  return shard_finish(shape, params, n_ctx, world, bounds, static_cast<const float*>(msgs), state, out,
                      static_cast<cudaStream_t>(stream));
}

int a2ats_decode_step_sharded(const a2ats_shape* shape, const a2ats_params* params, int32_t n_ctx, int32_t world,
                              int32_t rank, const int32_t* bounds, const void* q, const void* k_cache,
                              const void* v_cache, uint16_t* codes, const void* codebook, const void* chat,
                              const float* nrm, void* state, float* out, int32_t* sel_out, void* ws,
                              size_t ws_bytes, a2ats_comm* comm, void* stream) {
  int rc = shard_common(shape, params, n_ctx, world, rank, bounds);
  if (rc) return rc;
  if (!out) return A2ATS_EINVAL;
  if ((world > 1 && !comm) || (comm && (comm->world != world || comm->rank != rank))) return A2ATS_EINVAL;
  if (comm && !nccl().ok) return A2ATS_ENCCL;
  const ShardWs W = shard_ws_layout(shape, params, world);
  if (!ws || ws_bytes < W.total) return A2ATS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* msg = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + W.msg);
  float* recv = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + W.recv);
  // one rank: the attention writes the normalised output itself; only the state update follows
  rc = shard_partial(shape, params, n_ctx, world, rank, bounds, q, k_cache, v_cache, codes, codebook, chat, nrm,
                     state, msg, sel_out, ws, ws_bytes, st, world == 1 ? out : nullptr);
  if (rc) return rc;
  const size_t mf = msg_floats(shape);
  if (world > 1) {  // the step's only collective: every rank's partial and the new token's code
    if (nccl().all_gather(msg, recv, mf, kNcclFloat32, comm->nccl_comm, st) != 0) return A2ATS_ENCCL;
  } else {
    recv = msg;
  }
  return shard_finish(shape, params, n_ctx, world, bounds, recv, state, out, st, world > 1);
}

int a2ats_combine(const a2ats_shape* shape, int32_t nparts, const float* partials, float* out, void* stream) {
  int rc = check_shape(shape);
  if (rc) return rc;
  if (nparts < 1 || !partials || !out) return A2ATS_EINVAL;
  const size_t rows = (size_t)shape->B * shape->Hq;
  return cuda_status(launch_combine(partials, nparts, (int)rows, rows * 130, out, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
