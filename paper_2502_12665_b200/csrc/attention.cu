// a5 + a6: exact softmax attention over Sel = Sinks u TopK u Window
// (Eq. 2) with WRoPE logits (Eq. 11):
//   sinks / top-K rows : u_j = q~ . k_j          (bridge rotation R_b)
//   window rows        : u_j = (q R_{i-j}) . k_j = sum_m cos(r f_m) A_m + sin(r f_m) B_m,
//                        A_m = q_m k_m + q_{m+64} k_{m+64}, B_m = q_m k_{m+64} - q_{m+64} k_m
//                        (the relative identity of Eq. 3 applied to the query only).
//
// HBM-bound gather: every selected K/V row (2 x 256 B, scattered) is read once
// and shared by the G query heads of the GQA group.  One CTA = (row split,
// pair); 8 warps (one CTA per SM); a warp owns 16-row tiles.  Rows are gathered with cp.async
// (16 B pieces, XOR-swizzled so ldmatrix is conflict-free) into a warp-private
// ring of kStages tiles.  The per-tile contractions S = K_tile Q~^T (16 rows x
// G heads x 128) and O^T += V_tile^T P (128 x G x 16) use mma.sync m16n8k16
// (bf16 in, fp32 accumulate) only to keep the issue rate far below the memory
// rate; q~ and P are split hi + lo into two bf16 halves so both products carry
// fp32-level accuracy (~2^-16).  Window tiles compute their logits on FP32
// CUDA cores (the rotation differs per row).  fp32 online softmax in base 2;
// partial (m, l, o) per split; the last CTA of a pair combines the splits in
// fixed order (deterministic LSE combine, a6).
#include "internal.cuh"
#include "umma.cuh"

namespace a2ats {

namespace {
A2ATS_TL_DECL(g_attn_tl)
constexpr int kStages = 3;
constexpr int kTileBytes = 16 * 256;           // one K (or V) tile: 16 rows x 256 B
constexpr int kStageBytes = 2 * kTileBytes;    // K + V

struct SmemLayout {
  int tok, ring, q, sS, bcs, sW, red, total;
};
// NW warps per CTA: 8 (one CTA per SM) or 4 (two per SM, for grids of many (pair, split)
// work items: one CTA's prologue overlaps the other's stream)
template <int NW>
__host__ __device__ inline SmemLayout attn_smem(int R) {
  constexpr int kWarps = NW;
  SmemLayout s;
  s.tok = 0;
  s.ring = ((R * 4) + 127) / 128 * 128;
  s.q = s.ring + kWarps * kStages * kStageBytes;     // raw q (scaled) [8][128] fp32 for window tiles
  s.sS = s.q + 8 * kD * 4;                           // window logits [4 warps][16 rows][8 heads]
  s.bcs = s.sS + kWarps * 16 * 8 * 4;                // bridge (cos, sin) [64] float2
  s.sW = s.bcs + kHalf * 8;                          // precomputed window logits [64 rows][8 heads]
  s.red = s.ring;                                    // warp partials [4][8 heads][130], after the ring is dead
  s.total = s.sW + kWinPre * 8 * 4;
  return s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(uint16_t lo, uint16_t hi) { return lo | (uint32_t(hi) << 16); }
__device__ __forceinline__ void split_pair(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  uint16_t h0, l0, h1, l1;
  umma::split_bf16(x0, h0, l0);
  umma::split_bf16(x1, h1, l1);
  hi = pack_bf16(h0, h1);
  lo = pack_bf16(l0, l1);
}
// byte offset of (row, 16-B chunk) inside a 16 x 256 B tile, XOR swizzle on the chunk
__device__ __forceinline__ uint32_t swz(int row, int chunk) { return row * 256 + ((chunk ^ (row & 7)) << 4); }

template <int NW>
__device__ __forceinline__ void attn_body(const AttnArgs& a) {
  constexpr int kWarps = NW;
  constexpr int kThreads = NW * 32;
  extern __shared__ __align__(128) uint8_t smraw[];
  const SmemLayout SL = attn_smem<NW>(a.R);
  int32_t* s_tok = reinterpret_cast<int32_t*>(smraw + SL.tok);
  float* sQ = reinterpret_cast<float*>(smraw + SL.q);
  float* red = reinterpret_cast<float*>(smraw + SL.red);

  const int split = blockIdx.x, pair = blockIdx.y;
  const int b = pair / a.Hkv, h = pair - b * a.Hkv;
  const int G = a.G;
  const int hq0 = h * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g8 = lane >> 2, t4 = lane & 3;  // mma fragment coordinates

  // step inputs only, before the dependency wait: the query, fp32 and scaled to the base-2
  // logit domain, in smem (one 16-B load per thread) -- read by the window path -- and
  // q~ = q R_b (Eq. 12) as the mma B operand: head n = g8, d = 16kk + 2t4 + {0,1} (+8);
  // the lane's d and d + 64 sit in fragments kk and kk + 4, so it rotates its own pairs
  uint32_t qh[8][2], ql[8][2];
  {
    float2* sbcs = reinterpret_cast<float2*>(smraw + SL.bcs);
    if (tid < kHalf) sbcs[tid] = a.bcs[tid];
    if (tid < 128) {
      const int g = tid >> 4, e0 = (tid & 15) * 8;
      uint4 x = make_uint4(0, 0, 0, 0);
      if (g < G) x = ld_nc_u4(a.q + ((size_t)b * a.Hq + hq0 + g) * kD + e0);
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
      float4* d = reinterpret_cast<float4*>(sQ + g * kD + e0);
      d[0] = make_float4(bf_lo(w[0]) * a.scale_log2, bf_hi(w[0]) * a.scale_log2, bf_lo(w[1]) * a.scale_log2,
                         bf_hi(w[1]) * a.scale_log2);
      d[1] = make_float4(bf_lo(w[2]) * a.scale_log2, bf_hi(w[2]) * a.scale_log2, bf_lo(w[3]) * a.scale_log2,
                         bf_hi(w[3]) * a.scale_log2);
    }
    __syncthreads();
    const float* qs = sQ + g8 * kD;  // heads >= G hold zeros
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int d0 = kk * 16 + 2 * t4 + 8 * hf;
        const float2 x1 = *reinterpret_cast<const float2*>(qs + d0);
        const float2 x2 = *reinterpret_cast<const float2*>(qs + d0 + kHalf);
        const float2 c0 = sbcs[d0], c1 = sbcs[d0 + 1];
        split_pair(fmaf(x1.x, c0.x, -x2.x * c0.y), fmaf(x1.y, c1.x, -x2.y * c1.y), qh[kk][hf], ql[kk][hf]);
        split_pair(fmaf(x2.x, c0.x, x1.x * c0.y), fmaf(x2.y, c1.x, x1.y * c1.y), qh[kk + 4][hf], ql[kk + 4][hf]);
      }
  }
  const uint8_t* kbase = reinterpret_cast<const uint8_t*>(a.kc) + (size_t)pair * a.n_max * 256;
  const uint8_t* vbase = reinterpret_cast<const uint8_t*>(a.vc) + (size_t)pair * a.n_max * 256;
  float* sW = reinterpret_cast<float*>(smraw + SL.sW);
  // Window rows whose logits the prep kernel computed (wlog, rows j < n_wl of the window):
  // the split's leading window rows, whole tiles only unless the split ends first.
  auto load_wlog = [&](int keff_) {
    const int M_ = a.n_s + keff_ + a.n_w, p0_ = split * a.R, p1_ = min(p0_ + a.R, M_), pw_ = a.n_s + keff_;
    if (p0_ >= M_) return 0;
    const int jA = max(p0_, pw_) - pw_, nB_ = max(0, p1_ - max(p0_, pw_));
    const int c = max(0, min(nB_, a.n_wl - jA));
    const int npre = (c == nB_) ? nB_ : (c / 16) * 16;
    for (int k = tid; k < npre * 8; k += kThreads) sW[k] = __ldcg(a.wlog + ((size_t)pair * kWinPre + jA) * 8 + k);
    return npre;
  };
  // wlog comes from the prep kernel, two launches back when a select kernel runs in between
  // (complete when this grid starts); with keff == 0 no select is launched, and long-context /
  // posting-list selects write wlog themselves: read after the wait
  const bool wlog_early = !a.nsel && a.keff > 0 && !a.wlog_late;
  int nwpre = 0;
  if (wlog_early) nwpre = load_wlog(a.keff);
  pdl_wait();  // sel / counts come from select
  pdl_trigger();

  // Sel list of this pair on this rank: [sinks][top-K rows][window rows], ascending
  const int keff = a.nsel ? __ldcg(a.nsel + pair) : a.keff;
  if (!wlog_early) nwpre = load_wlog(keff);
  const int M = a.n_s + keff + a.n_w;
  const int nsplit = (M + a.R - 1) / a.R;
  if (M == 0) {  // no row of this pair lives on this rank: empty partial (sharded mode only)
    if (split == 0 && a.part_out) {
      for (int i = tid; i < G * 130; i += kThreads) {
        const int gg = i / 130, f = i - gg * 130;
        a.part_out[((size_t)b * a.Hq + hq0 + gg) * 130 + f] = (f == 0) ? -INFINITY : 0.f;
      }
    }
    return;
  }
  if (split >= nsplit) return;
  const int p0 = split * a.R, p1 = min(p0 + a.R, M);
  const int pw = a.n_s + keff;               // first window position in the Sel list
  const int pwc = a.win_as_bridge ? M : pw;  // first row with a per-row (window) rotation
  const int nA = max(0, min(p1, pwc) - p0);  // bridge rows of this split
  const int nB = (p1 - p0) - nA;             // window rows of this split
  const int gA = (nA + 15) >> 4, gB = (nB + 15) >> 4, ngroups = gA + gB;

  for (int i0 = 0; i0 < p1 - p0; i0 += 8 * kThreads) {  // 8 index loads in flight per thread
    int tv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int p = p0 + i0 + j * kThreads + tid;
      tv[j] = 0;
      if (p < p1) {  // local row index of the K/V arrays
        if (p < a.n_s) tv[j] = a.sink_lo + p - a.shard_begin;
        else if (p < pw) tv[j] = __ldcg(a.sel + (size_t)pair * a.sel_stride + (p - a.n_s)) - a.shard_begin;
        else tv[j] = a.win_lo + (p - pw) - a.shard_begin;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (p0 + i0 + j * kThreads + tid < p1) s_tok[i0 + j * kThreads + tid] = tv[j];
  }
  A2ATS_TL(g_attn_tl, 2);
  __syncthreads();

  uint8_t* wring = smraw + SL.ring + warp * (kStages * kStageBytes);
  const uint32_t wring_s = smem_u32(wring);

  // tile g of this warp's sequence -> (first local row, row count, is window).  Window
  // tiles come first: their FP32 logits then overlap the ring's loads of later tiles.
  auto tile_of = [&](int g, int& r0, int& nr) -> bool {
    if (g < gB) {
      r0 = nA + g * 16;
      nr = min(16, nA + nB - r0);
      return true;
    }
    r0 = (g - gB) * 16;
    nr = min(16, nA - r0);
    return false;
  };
  auto issue = [&](int s) {
    const int g = s * kWarps + warp;
    if (g < ngroups) {
      int r0, nr;
      const bool win = tile_of(g, r0, nr);
      uint8_t* st = wring + (s % kStages) * kStageBytes;
      if (win && r0 - nA >= nwpre) {  // warm L1 with this lane's (cos, sin) row half for the window logits
        const int row = lane >> 1, rr = row < nr ? row : nr - 1;
        const float2* p = a.cs + (size_t)(a.n_ctx - 1 - a.shard_begin - s_tok[r0 + rr]) * kHalf + (lane & 1) * 32;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 16));
      }
      // piece idx = lane + 32 i: (kv = i >> 3, row = (lane >> 4) + 2 (i & 7), chunk = lane & 15);
      // the lane's 8 rows are read from s_tok once, all loads before the first use
      const int chunk = lane & 15;
      uint32_t roff[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int row = (lane >> 4) + 2 * j;
        roff[j] = (uint32_t)s_tok[r0 + (row < nr ? row : nr - 1)];  // pad rows re-read a valid row
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int kv = i >> 3, row = (lane >> 4) + 2 * (i & 7);
        const size_t off = (size_t)roff[i & 7] * 256 + chunk * 16;
        cp_async16(st + kv * kTileBytes + swz(row, chunk), (kv ? vbase : kbase) + off);
      }
    }
    cp_async_commit();
  };

  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrun0 = -INFINITY, mrun1 = -INFINITY, lrun0 = 0.f, lrun1 = 0.f;  // heads 2*t4, 2*t4+1

  const int nsteps = (ngroups > warp) ? (ngroups - warp + kWarps - 1) / kWarps : 0;
#pragma unroll 1
  for (int s = 0; s < kStages - 1; ++s) issue(s);
  const int icur = a.n_ctx - 1 - a.shard_begin;  // current token, in local row units
  float* sS = reinterpret_cast<float*>(smraw + SL.sS) + warp * 128;

#pragma unroll 1
  for (int s = 0; s < nsteps; ++s) {
    issue(s + kStages - 1);
    cp_async_wait<kStages - 1>();
    __syncwarp();
    const int g = s * kWarps + warp;
    int r0, nr;
    const bool win = tile_of(g, r0, nr);
    const uint32_t kst = wring_s + (s % kStages) * kStageBytes;
    const uint32_t vst = kst + kTileBytes;
    const int mi = lane >> 3, rr = lane & 7;

    float sc[4];
    if (!win) {
      // four independent accumulation chains (hi / lo x even / odd kk), summed at the end
      float ca[4] = {0.f, 0.f, 0.f, 0.f}, cb[4] = {0.f, 0.f, 0.f, 0.f};
      float cc[4] = {0.f, 0.f, 0.f, 0.f}, cd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < 8; kk += 2) {
        uint32_t af0[4], af1[4];
        ldsm_x4(kst + swz(rr + 8 * (mi & 1), 2 * kk + (mi >> 1)), af0);
        ldsm_x4(kst + swz(rr + 8 * (mi & 1), 2 * (kk + 1) + (mi >> 1)), af1);
        mma16816(ca, af0, qh[kk][0], qh[kk][1]);
        mma16816(cb, af1, qh[kk + 1][0], qh[kk + 1][1]);
        mma16816(cc, af0, ql[kk][0], ql[kk][1]);
        mma16816(cd, af1, ql[kk + 1][0], ql[kk + 1][1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) sc[i] = (ca[i] + cb[i]) + (cc[i] + cd[i]);
    } else if (r0 - nA < nwpre) {  // window rows with precomputed logits
      const float* w = sW + (r0 - nA) * 8 + 2 * t4;
      sc[0] = w[g8 * 8];
      sc[1] = w[g8 * 8 + 1];
      sc[2] = w[(g8 + 8) * 8];
      sc[3] = w[(g8 + 8) * 8 + 1];
    } else {
      // further window rows: exact relative rotation per row on FP32 cores (lane = row, half of the pairs)
      const int row = lane >> 1, hf = lane & 1;
      const int rrow = row < nr ? row : nr - 1;
      const int r = icur - s_tok[r0 + rrow];
      const float4* csp = reinterpret_cast<const float4*>(a.cs + (size_t)r * kHalf + hf * 32);
      const uint8_t* krow = wring + (s % kStages) * kStageBytes;
      // c (8-pair chunk) outer and rolled; per chunk the k and (cos, sin) loads are issued
      // together, then every head of the group accumulates (heads unrolled up to 8)
      float acc[8];
#pragma unroll
      for (int gg = 0; gg < 8; ++gg) acc[gg] = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {  // m = hf*32 + c*8 + i
        const uint4 k1 = *reinterpret_cast<const uint4*>(krow + swz(row, hf * 4 + c));
        const uint4 k2 = *reinterpret_cast<const uint4*>(krow + swz(row, 8 + hf * 4 + c));
        float4 t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = __ldg(csp + c * 4 + j);
        const uint32_t w1[4] = {k1.x, k1.y, k1.z, k1.w}, w2[4] = {k2.x, k2.y, k2.z, k2.w};
        const float* qa = sQ + hf * 32 + c * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float ka = (i & 1) ? bf_hi(w1[i >> 1]) : bf_lo(w1[i >> 1]);
          const float kb = (i & 1) ? bf_hi(w2[i >> 1]) : bf_lo(w2[i >> 1]);
          const float cv = (i & 1) ? t[i >> 1].z : t[i >> 1].x, sv = (i & 1) ? t[i >> 1].w : t[i >> 1].y;
#pragma unroll
          for (int gg = 0; gg < 8; ++gg) {
            if (gg < G) {
              const float q1 = qa[gg * kD + i], q2 = qa[gg * kD + i + kHalf];
              acc[gg] = fmaf(cv, fmaf(q1, ka, q2 * kb), fmaf(sv, fmaf(q1, kb, -q2 * ka), acc[gg]));
            }
          }
        }
      }
#pragma unroll
      for (int gg = 0; gg < 8; ++gg) {
        const float v = acc[gg] + __shfl_xor_sync(0xffffffffu, acc[gg], 1);
        if (hf == 0) sS[row * 8 + gg] = v;  // heads >= G: 0
      }
      __syncwarp();
      sc[0] = sS[g8 * 8 + 2 * t4];
      sc[1] = sS[g8 * 8 + 2 * t4 + 1];
      sc[2] = sS[(g8 + 8) * 8 + 2 * t4];
      sc[3] = sS[(g8 + 8) * 8 + 2 * t4 + 1];
    }
    // mask pad rows of the tile
    if (g8 >= nr) sc[0] = sc[1] = -INFINITY;
    if (g8 + 8 >= nr) sc[2] = sc[3] = -INFINITY;

    // online softmax per head (heads 2*t4, 2*t4+1); rows spread over lanes with equal t4
    float mx0 = fmaxf(sc[0], sc[2]), mx1 = fmaxf(sc[1], sc[3]);
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float mn0 = fmaxf(mrun0, mx0), mn1 = fmaxf(mrun1, mx1);  // finite: every tile has >= 1 row
    const float sc0 = exp2f(mrun0 - mn0), sc1 = exp2f(mrun1 - mn1);
    mrun0 = mn0;
    mrun1 = mn1;
    const float p0 = exp2f(sc[0] - mn0), p1 = exp2f(sc[1] - mn1);
    const float p2 = exp2f(sc[2] - mn0), p3 = exp2f(sc[3] - mn1);
    lrun0 = lrun0 * sc0 + p0 + p2;
    lrun1 = lrun1 * sc1 + p1 + p3;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i][0] *= sc0;
      o[i][1] *= sc1;
      o[i][2] *= sc0;
      o[i][3] *= sc1;
    }
    uint32_t ph0, pl0, ph1, pl1;
    split_pair(p0, p1, ph0, pl0);  // rows g8:   heads (2t4, 2t4+1)
    split_pair(p2, p3, ph1, pl1);  // rows g8+8
    const uint32_t bh0 = movm_t(ph0), bh1 = movm_t(ph1), bl0 = movm_t(pl0), bl1 = movm_t(pl1);
#pragma unroll
    for (int ds = 0; ds < 8; ++ds) {
      uint32_t af[4];
      ldsm_x4_t(vst + swz(rr + 8 * (mi >> 1), 2 * ds + (mi & 1)), af);
      mma16816(o[ds], af, bh0, bh1);
      mma16816(o[ds], af, bl0, bl1);
    }
    __syncwarp();  // every lane done with this ring slot before it is refilled
  }
  A2ATS_TL(g_attn_tl, 3);
  cp_async_wait<0>();
  __syncthreads();  // all warps out of the ring: it is reused for the warp partials

  // per-warp partial: l summed over rows (lanes with equal t4)
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    lrun0 += __shfl_xor_sync(0xffffffffu, lrun0, off);
    lrun1 += __shfl_xor_sync(0xffffffffu, lrun1, off);
  }
  {
    float* r0p = red + (warp * 8 + 2 * t4) * 130;
    float* r1p = red + (warp * 8 + 2 * t4 + 1) * 130;
    if (g8 == 0) {
      r0p[0] = mrun0; r0p[1] = lrun0;
      r1p[0] = mrun1; r1p[1] = lrun1;
    }
#pragma unroll
    for (int ds = 0; ds < 8; ++ds) {
      r0p[2 + ds * 16 + g8] = o[ds][0];
      r1p[2 + ds * 16 + g8] = o[ds][1];
      r0p[2 + ds * 16 + g8 + 8] = o[ds][2];
      r1p[2 + ds * 16 + g8 + 8] = o[ds][3];
    }
  }
  __syncthreads();

  // combine the warps: thread tid -> element e = tid % 128 of heads tid / 128, + 2, ...
  const int e = tid & (kD - 1), gsel = tid >> 7;
  // final result of a pair: normalised output, or (sharded mode) the rank's partial
  // (m, l, o) in the base-2 logit domain for the cross-rank LSE combine
  auto emit = [&](int gg, float M, float den, float num) {
    if (a.part_out) {
      float* dst = a.part_out + ((size_t)b * a.Hq + hq0 + gg) * 130;
      dst[2 + e] = num;
      if (e == 0) {
        dst[0] = M;
        dst[1] = den;
      }
    } else {
      a.out[((size_t)b * a.Hq + hq0 + gg) * kD + e] = num / den;
    }
  };
  float* part = a.part + (size_t)pair * G * a.nsplit * 130;  // stride: max splits
  const bool single = (nsplit == 1);
  for (int gg = gsel; gg < G; gg += kThreads / kD) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, red[(w * 8 + gg) * 130]);
    float acc = 0.f, den = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float mw = red[(w * 8 + gg) * 130];
      const float sw = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      acc = fmaf(red[(w * 8 + gg) * 130 + 2 + e], sw, acc);
      den = fmaf(red[(w * 8 + gg) * 130 + 1], sw, den);
    }
    if (single) {
      emit(gg, M, den, acc);
    } else {
      float* dst = part + ((size_t)gg * a.nsplit + split) * 130;
      dst[2 + e] = acc;
      if (e == 0) {
        dst[0] = M;
        dst[1] = den;
      }
    }
  }
  if (single) return;

  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(a.counter + pair, 1u);
    s_last = (prev == (unsigned)(nsplit - 1));
  }
  __syncthreads();
  if (!s_last) return;
  A2ATS_TL(g_attn_tl, 4);
  __threadfence();
  // (m, l) of every (head, split) into smem, one load per thread; then, per head, the
  // o values of all splits with their loads in flight together (fixed split order)
  float* sML = red;  // the warp partials are consumed
  for (int i = tid; i < G * nsplit; i += kThreads) {  // i = gg * nsplit + s; part stride is the max split count
    const float* src = part + ((size_t)(i / nsplit) * a.nsplit + i % nsplit) * 130;
    sML[2 * i] = __ldcg(src);
    sML[2 * i + 1] = __ldcg(src + 1);
  }
  __syncthreads();
#pragma unroll 1
  for (int gg = gsel; gg < G; gg += kThreads / kD) {
    const float* src = part + (size_t)gg * a.nsplit * 130 + 2 + e;
    const float* ml = sML + 2 * gg * nsplit;
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, ml[2 * s]);
    float num = 0.f, den = 0.f;
#pragma unroll 1
    for (int s0 = 0; s0 < nsplit; s0 += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (s0 + j < nsplit) ? __ldcg(src + (s0 + j) * 130) : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (s0 + j < nsplit) {
          const float ms = ml[2 * (s0 + j)];
          const float sw = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
          num = fmaf(v[j], sw, num);
          den = fmaf(ml[2 * (s0 + j) + 1], sw, den);
        }
      }
    }
    emit(gg, M, den, num);
  }
  if (tid == 0) a.counter[pair] = 0u;  // leave the workspace in its zero state
}

template <int NW>
__global__ __launch_bounds__(NW * 32, NW <= 4 ? 2 : 1) void attn_mma_kernel(AttnArgs a) {
  A2ATS_TL(g_attn_tl, 0);
  attn_body<NW>(a);
  A2ATS_TL(g_attn_tl, 1);
}

// Cross-rank log-sum-exp combine of partials (base-2 logits), fixed rank order; rank r's
// partials [rows][130] start at parts + r * stride.
__global__ void combine_kernel(const float* __restrict__ parts, int R, int rows, size_t stride,
                               float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x, e = threadIdx.x;
  if (row >= rows) return;
  float M = -INFINITY;
  for (int r = 0; r < R; ++r) M = fmaxf(M, parts[(size_t)r * stride + (size_t)row * 130]);
  float num = 0.f, den = 0.f;
  for (int r = 0; r < R; ++r) {
    const float* p = parts + (size_t)r * stride + (size_t)row * 130;
    const float sw = (p[0] == -INFINITY) ? 0.f : exp2f(p[0] - M);
    num = fmaf(p[2 + e], sw, num);
    den = fmaf(p[1], sw, den);
  }
  out[(size_t)row * kD + e] = num / den;
}
}  // namespace

template <int NW>
cudaError_t launch_attention_nw(const AttnArgs& a, int P, cudaStream_t st) {
  const SmemLayout L = attn_smem<NW>(a.R);
  cudaError_t e = ensure_smem(attn_mma_kernel<NW>, L.total);
  if (e != cudaSuccess) return e;
  dim3 grid(a.nsplit, P, 1);
  return launch_pdl(attn_mma_kernel<NW>, grid, dim3(NW * 32), L.total, st, a);
}

// 4-warp CTAs (two per SM) when the grid has at least two (pair, split) items per SM
// (measured at C4: 362 -> 350 us), 8-warp CTAs otherwise (C2: one CTA per pair is faster)
#ifndef A2ATS_ATTN_NW4
#define A2ATS_ATTN_NW4 0  // tuning builds only: 1 forces 4-warp CTAs
#endif
cudaError_t launch_attention(const AttnArgs& a, int P, int /*GT*/, cudaStream_t st) {
  if (A2ATS_ATTN_NW4 || (long long)P * a.nsplit >= 2LL * sm_count()) return launch_attention_nw<4>(a, P, st);
  return launch_attention_nw<8>(a, P, st);
}

cudaError_t launch_combine(const float* parts, int R, int rows, size_t stride, float* out, cudaStream_t st) {
  return launch_pdl(combine_kernel, dim3(rows), dim3(kD), 0, st, parts, R, rows, stride, out);
}

}  // namespace a2ats

A2ATS_TL_EXPORT(a2ats_debug_attn_timeline, a2ats::g_attn_tl)
