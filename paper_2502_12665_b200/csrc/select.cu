// a3 + a4: approximate scores through the code stream and exact top-K selection.
//
// Scores take only L distinct values per (b, KV head) pair (u^_t = LUT[s_t],
// Eq. 21), so the K-th largest score is found by a count-weighted
// selection over the L codewords, not over the N tokens.  One CTA owns one pair:
//
//  1. candidate counts per codeword: the caller-maintained hist minus the
//     sink/window codes, or (without hist) a pass over the candidate codes.  Both
//     read only step inputs, so they run before the dependency wait (overlapping
//     the LUT kernel), as does the prefetch of the first chunk of codes;
//  2. keys = ~ordered(agg) and their range; a weighted histogram over 256
//     equal-width value bins finds the bin holding the K-th token; its (few)
//     codewords are compacted and the exact K-th key v* is resolved by ranking
//     them (one thread per survivor; radix passes if there are very many); tie
//     quota m = K - #{agg > v*};
//  3. 2-bit class per codeword (1: agg > v*, 2: agg == v*), replicated 32x in
//     shared memory so lane l reads bank l (conflict-free gather by code);
//  4. stream the codes: each thread classifies 64 consecutive tokens, one block
//     scan gives every thread its output offset, and the selected indices are
//     written in ascending order.  A token with agg == v* is kept iff fewer than
//     m such tokens precede it: the lowest-index tie-break of reading Q12.
//
// The sequence-sharded step takes v*, m and this rank's tie
// share from replicated histograms (select_shard_thresh_kernel) and then runs the
// same persistent scan over the rank's local candidate range.
#include "internal.cuh"
#include "umma.cuh"

namespace a2ats {

namespace {
A2ATS_TL_DECL(g_sel_tl)
A2ATS_TL_DECL(g_selp_tl)  // postings kernel phase marks (tuning builds)
A2ATS_TL_DECL(g_selc_tl)
A2ATS_PHASE_DECL(g_sel_phase)

constexpr int kNT = 512;             // threads per CTA
constexpr int kNW = kNT / 32;
constexpr int kTPT = 64;             // consecutive tokens per thread per chunk
constexpr int kCH = kNT * kTPT;      // tokens per chunk (32768: 16-bit scan fields cannot carry)
constexpr int kSurvCap = 2048;       // survivor list capacity
constexpr int kRankMax = kNT;        // survivors ranked directly (one thread each)

// kFused: one CTA per pair does everything (contexts of one code chunk).  Long contexts
// split it: kThresh (per pair: counts, v*, m, compact class table to global) then kScanC
// (per (pair, chunk of 32768 tokens): classify, publish the chunk's counts, look back at
// the pair's earlier chunks for the output offsets, emit).
enum SelMode { kFused = 0, kThresh = 4, kScanC = 5 };

constexpr int kWinScratch = 32768 + 16384 + 8 * kD * 4;  // window logits scratch (threshold kernel)

template <int MODE>
struct ModeTraits {
  static constexpr bool surv = (MODE == kFused || MODE == kThresh);   // find_level
  static constexpr bool codes = (MODE == kFused || MODE == kScanC);   // code chunk
  static constexpr int extra = (MODE == kThresh) ? kWinScratch : 0;  // bytes after the survivors
  static constexpr int min_blocks = (MODE == kThresh || MODE == kScanC) ? 2 : 1;
};

// Thread group policy of the selection helpers (thread index and barrier): the whole CTA
struct CtaGrp {
  static __device__ __forceinline__ int tid() { return threadIdx.x; }
  static __device__ __forceinline__ void sync() { __syncthreads(); }
};

struct SelShared {
  int bins[256];
  uint32_t wsum[kNW];
  int s_digit, s_kk, s_nsurv, s_total;
  uint32_t s_kmin, s_kmax, s_kstar, s_m;
  int s_gt, s_eq;
  uint32_t s_before[2];
};

// cnt[l] = hist[l] - #(local sink/window tokens with code l)   (hist given)
//        = #(local candidate tokens with code l)                (otherwise)
// Step inputs only (hist, codes).
template <int NT = kNT, class Grp = CtaGrp>
__device__ void load_cnt(const SelArgs& a, int pair, int* cnt, const uint16_t* cp_local) {
  const int tid = Grp::tid();
  const int32_t* histp = a.hist ? a.hist + (size_t)pair * a.L : nullptr;
  const int lo = a.shard_begin, hi = a.shard_begin + a.shard_len;  // local global-index range
  if (histp) {
    for (int base = 0; base < a.L; base += 8 * NT) {  // all loads of a batch in flight before use
      int hv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int l = base + i * NT + tid;
        hv[i] = l < a.L ? __ldg(histp + l) : 0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int l = base + i * NT + tid;
        if (l < a.L) cnt[l] = hv[i];
      }
    }
    Grp::sync();
    // remove the local sinks [0, n_s) and window [w0, n_ctx): they are not candidates
    // (append: hist does not hold token n_ctx - 1 yet, whose code the prep kernel computes;
    // deferred a0: nor the newest hist_lag tokens)
    const int nrem = a.n_s + max(0, a.hist_end - a.w0);
    for (int i = tid; i < nrem; i += NT) {
      const int t = i < a.n_s ? i : a.w0 + (i - a.n_s);
      if (t >= lo && t < hi) atomicSub(&cnt[cp_local[t - lo]], 1);
    }
  } else {
    for (int l = tid; l < a.L; l += NT) cnt[l] = 0;
    Grp::sync();
    const int c0 = max(a.c0, lo), c1 = min(a.c1, hi);
    if (c0 < c1) {
      const int v0 = (c0 - lo) >> 3, v1 = (c1 - lo + 7) >> 3;
      for (int vi = v0 + tid; vi < v1; vi += NT) {
        const uint4 x = ld_nc_u4(cp_local + (size_t)vi * 8);
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int t = lo + vi * 8 + e;
          if (t >= c0 && t < c1) atomicAdd(&cnt[(w[e >> 1] >> ((e & 1) * 16)) & 0xffffu], 1);
        }
      }
    }
  }
  Grp::sync();
}

// key[l] = ~ordered(agg[l]) (ascending key = descending agg) and the key range of the
// codewords with cnt > 0 -> S.s_kmin / S.s_kmax.  Needs cnt (synced); ends synced.
template <int NT = kNT, class Grp = CtaGrp>
__device__ void load_keys(const SelArgs& a, SelShared& S, int pair, const int* cnt, uint32_t* key) {
  const int tid = Grp::tid(), lane = tid & 31;
  const float* aggp = a.agg + (size_t)pair * a.L;
  if (tid == 0) {
    S.s_kmin = 0xffffffffu;
    S.s_kmax = 0u;
  }
  uint32_t kmn = 0xffffffffu, kmx = 0u;
  for (int base = 0; base < a.L; base += 8 * NT) {
    float av[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int l = base + i * NT + tid;
      av[i] = l < a.L ? __ldcg(aggp + l) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int l = base + i * NT + tid;
      if (l < a.L) {
        const uint32_t k = ~ordered_key(av[i]);
        key[l] = k;
        if (cnt[l] > 0) {
          kmn = min(kmn, k);
          kmx = max(kmx, k);
        }
      }
    }
  }
  kmn = __reduce_min_sync(0xffffffffu, kmn);
  kmx = __reduce_max_sync(0xffffffffu, kmx);
  Grp::sync();  // s_kmin / s_kmax initialised
  if (lane == 0) {
    atomicMin(&S.s_kmin, kmn);
    atomicMax(&S.s_kmax, kmx);
  }
  Grp::sync();
}

// Warp 0: find the digit of bins[] that holds rank kk (1-based); writes s_digit, s_kk.
__device__ __forceinline__ void pick_digit(SelShared& S, int kk) {
  const int lane = threadIdx.x & 31;
  int loc[8], s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    loc[i] = S.bins[lane * 8 + i];
    s += loc[i];
  }
  int incl = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  const int excl = incl - s;
  const unsigned hit = __ballot_sync(0xffffffffu, excl < kk && kk <= incl);
  if (lane == __ffs(hit) - 1) {
    int c = excl;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (c + loc[i] >= kk) {
        S.s_digit = lane * 8 + i;
        S.s_kk = kk - c;
        break;
      }
      c += loc[i];
    }
  }
  __syncwarp();
}

// Count-weighted selection of the keff-th smallest key over cnt / key (all threads),
// given the key range S.s_kmin..S.s_kmax.  Result in S.s_kstar (key of v*) and
// S.s_m (tie quota, >= 1).
template <int NT = kNT, int SC = kSurvCap, class Grp = CtaGrp>
__device__ void find_level(const SelArgs& a, SelShared& S, const int* cnt, const uint32_t* key, int keff,
                           uint32_t* skey, int* scnt) {
  const int tid = Grp::tid(), lane = tid & 31, warp = tid >> 5;
  const uint32_t kmn = S.s_kmin, kmx = S.s_kmax;
  if (kmn == kmx) {  // a single level holds every candidate
    if (tid == 0) {
      S.s_kstar = kmn;
      S.s_m = (uint32_t)keff;
    }
    Grp::sync();
    return;
  }
  for (int i = tid; i < 256; i += NT) S.bins[i] = 0;
  if (tid == 0) S.s_nsurv = 0;
  Grp::sync();
  // 256 bins of equal width in agg VALUE over [amin, amax], ascending bin = descending
  // agg (monotone and deterministic: one subtract, one multiply, one truncation).
  auto key_val = [](uint32_t k) {
    const uint32_t o = ~k;  // ordered key
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
  };
  const float amax = key_val(kmn), amin = key_val(kmx);
  const float scale = 255.99f / (amax - amin);
  auto bin_of = [&](uint32_t k) {
    const float d = amax - key_val(k);
    return d > 0.f ? min(255, (int)(d * scale)) : 0;
  };
  for (int l = tid; l < a.L; l += NT) {
    const int c = cnt[l];
    if (c > 0) atomicAdd(&S.bins[bin_of(key[l])], c);
  }
  Grp::sync();
  if (warp == 0) pick_digit(S, keff);
  Grp::sync();
  A2ATS_PHASE(g_sel_phase, 3);
  if (NT == 256 && tid == 0) A2ATS_TLX(g_sel_tl, 6);
  const int bstar = S.s_digit;
  int kk = S.s_kk;
  // survivors = candidate codewords of bin b*, one pass (order is irrelevant below)
  if (a.L <= 32 * NT) {  // keep flags per thread in a mask, one block scan for the slots
    uint32_t kmask = 0u;
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      const int l = i * NT + tid;
      if (l < a.L && cnt[l] > 0 && bin_of(key[l]) == bstar) kmask |= 1u << i;
    }
    const int nk = __popc(kmask);
    int incl = nk;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) S.wsum[warp] = (uint32_t)incl;
    Grp::sync();
    int base = incl - nk, tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
      const int v = (int)S.wsum[w];
      base += (w < warp) ? v : 0;
      tot += v;
    }
    while (kmask) {
      const int i = __ffs(kmask) - 1;
      kmask &= kmask - 1u;
      const int l = i * NT + tid;
      if (base < SC) {
        skey[base] = key[l];
        scnt[base] = cnt[l];
      }
      ++base;
    }
    if (tid == 0) S.s_nsurv = tot;
  } else
  for (int l0 = 0; l0 < a.L; l0 += NT) {
    const int l = l0 + tid;
    const bool keep = l < a.L && cnt[l] > 0 && bin_of(key[l]) == bstar;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (bal) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&S.s_nsurv, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int slot = base + __popc(bal & ((1u << lane) - 1u));
      if (keep && slot < SC) {
        skey[slot] = key[l];
        scnt[slot] = cnt[l];
      }
    }
  }
  Grp::sync();
  A2ATS_PHASE(g_sel_phase, 4);
  if (NT == 256 && tid == 0) A2ATS_TLX(g_sel_tl, 7);
  const int nsurv = S.s_nsurv;
  if (nsurv <= NT) {
    // rank each survivor directly: v* is the key with #(< v*) < kk <= #(<= v*);
    // equal keys write equal values
    if (tid < nsurv) {
      const uint32_t ki = skey[tid];
      int less = 0, leq = 0;
#pragma unroll 4
      for (int j = 0; j < nsurv; ++j) {
        const uint32_t kj = skey[j];
        const int cj = scnt[j];
        less += (kj < ki) ? cj : 0;
        leq += (kj <= ki) ? cj : 0;
      }
      if (less < kk && kk <= leq) {
        S.s_kstar = ki;
        S.s_m = (uint32_t)(kk - less);
      }
    }
    Grp::sync();
    return;
  }
  if (nsurv <= SC) {
    if (warp == 0) {
      // exact K-th key among the survivors: radix passes from their first differing bit
      uint32_t sa = 0xffffffffu, so = 0u;
      for (int i = lane; i < nsurv; i += 32) {
        sa &= skey[i];
        so |= skey[i];
      }
      sa = __reduce_and_sync(0xffffffffu, sa);
      so = __reduce_or_sync(0xffffffffu, so);
      const uint32_t diff = sa ^ so;
      uint32_t prefix = sa, mask = 0xffffffffu;
      if (diff) {
        const int top = 31 - __clz(diff);
        mask = (top >= 31) ? 0u : ~((2u << top) - 1u);
        prefix = sa & mask;
        for (int pass = top / 8; pass >= 0; --pass) {
          const int shift = 8 * pass;
          for (int i = lane; i < 256; i += 32) S.bins[i] = 0;
          __syncwarp();
          for (int i = lane; i < nsurv; i += 32) {
            const uint32_t k = skey[i];
            if ((k & mask) == prefix) atomicAdd(&S.bins[(k >> shift) & 255u], scnt[i]);
          }
          __syncwarp();
          pick_digit(S, kk);
          prefix = (prefix & ~(0xffu << shift)) | ((uint32_t)S.s_digit << shift);
          mask |= 0xffu << shift;
          kk = S.s_kk;
        }
      }
      if (lane == 0) {
        S.s_kstar = prefix;
        S.s_m = (uint32_t)kk;
      }
    }
    Grp::sync();
    return;
  }
  // degenerate value distributions (more survivors than the list holds): block-wide
  // byte passes restricted to bin b*
  uint32_t prefix = 0, mask = 0;
  for (int pass = 3; pass >= 0; --pass) {
    const int shift = 8 * pass;
    for (int i = tid; i < 256; i += NT) S.bins[i] = 0;
    Grp::sync();
    for (int l = tid; l < a.L; l += NT) {
      const int c = cnt[l];
      const uint32_t k = key[l];
      if (c > 0 && bin_of(k) == bstar && (k & mask) == prefix) atomicAdd(&S.bins[(k >> shift) & 255u], c);
    }
    Grp::sync();
    if (warp == 0) pick_digit(S, kk);
    Grp::sync();
    prefix |= (uint32_t)S.s_digit << shift;
    mask |= 0xffu << shift;
    kk = S.s_kk;
  }
  if (tid == 0) {
    S.s_kstar = prefix;
    S.s_m = (uint32_t)kk;
  }
  Grp::sync();
}

// 2-bit classes vs kstar, replicated 32x into tbl[word * 32 + replica] (tbl may alias
// key / cnt: every word is computed into registers before the first write).  One
// thread per word (W <= 1024); the 16-B chunks are visited in a per-thread rotated
// order so a quarter-warp touches distinct banks.
template <int NT = kNT>
__device__ void build_table(const SelArgs& a, const uint32_t* key, uint32_t kstar, uint32_t* tbl) {
  const int tid = threadIdx.x;
  constexpr int kMaxItems = 1024 / NT;  // words tid, tid + NT, ... (W <= 1024)
  uint32_t word[kMaxItems];
#pragma unroll
  for (int j = 0; j < kMaxItems; ++j) {
    const int w = j * NT + tid;
    uint32_t x = 0;
    if (w < a.W) {
      if (w * 16 + 16 <= a.L) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int qq = (q + w) & 3;
          const uint4 k4 = *reinterpret_cast<const uint4*>(key + w * 16 + 4 * qq);
          const uint32_t kv[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t c = (kv[e] < kstar) ? 1u : ((kv[e] == kstar) ? 2u : 0u);
            x |= c << (2 * (4 * qq + e));
          }
        }
      } else {
#pragma unroll 1
        for (int e = 0; e < 16 && w * 16 + e < a.L; ++e) {
          const uint32_t k = key[w * 16 + e];
          x |= ((k < kstar) ? 1u : ((k == kstar) ? 2u : 0u)) << (2 * e);
        }
      }
    }
    word[j] = x;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kMaxItems; ++j) {
    const int w = j * NT + tid;
    if (w < a.W) {
      uint4* dst = reinterpret_cast<uint4*>(tbl + w * 32);
      const uint4 v = make_uint4(word[j], word[j], word[j], word[j]);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[(q + w) & 7] = v;
    }
  }
  __syncthreads();
}

// cp.async one chunk of local codes into sC: coalesced 16-B global pieces; thread t's
// 8 pieces (its 64 consecutive tokens) land at t*8 + (i ^ (t & 7)) (conflict-free reads).
__device__ __forceinline__ void prefetch_chunk(const SelArgs& a, const uint16_t* cp_local, int cb, int c1, uint4* sC) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lo = a.shard_begin;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int u = j * 32 + lane;                   // piece within the warp's 256
    const int owner = warp * 32 + (u >> 3), i = u & 7;
    const int t0 = cb + (warp * 256 + u) * 8;      // first token of the piece (global index)
    uint4* dst = sC + owner * 8 + (i ^ (owner & 7));
    if (t0 < c1) cp_async16(dst, cp_local + (t0 - lo));
    else *dst = make_uint4(0, 0, 0, 0);  // codes past the range must be valid (< L)
  }
  cp_async_commit();
}

__device__ __forceinline__ uint32_t span_mask(int lo, int hi) {  // 2-bit fields [lo, hi) of 16
  lo = max(lo, 0);
  hi = min(hi, 16);
  if (hi <= lo) return 0u;
  const uint32_t mh = hi >= 16 ? 0xffffffffu : ((1u << (2 * hi)) - 1u);
  const uint32_t ml = (1u << (2 * lo)) - 1u;
  return mh & ~ml;
}

// Stream the local candidate codes (first chunk already prefetched into sC) and emit
// the selected global token indices in ascending order: every token above v*, plus
// the first m tied tokens.  Returns the number emitted.
__device__ uint32_t scan_emit(const SelArgs& a, SelShared& S, const uint32_t* tbl, const uint16_t* cp_local, int c0,
                              int c1, uint32_t m, uint32_t cap, int32_t* selp, uint4* sC) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lo = a.shard_begin;
  const int first = lo + (((c0 - lo) >> 3) << 3);  // 8-aligned (local index) start
  const int nchunk = c1 > c0 ? (c1 - first + kCH - 1) / kCH : 0;
  uint32_t run_gt = 0, run_eq = 0;
#pragma unroll 1
  for (int ch = 0; ch < nchunk; ++ch) {
    const int cb = first + ch * kCH;
    cp_async_wait<0>();
    __syncthreads();  // this chunk is in sC; the previous chunk is fully consumed
    A2ATS_PHASE(g_sel_phase, 8);
    const int t0 = cb + tid * kTPT;
    // classify the thread's 64 tokens, 16 per pass (rolled: straight-line code of this
    // size stalls on instruction fetch); p0..p3 = passes 0..3 after the register shift
    uint32_t p0 = 0u, p1 = 0u, p2 = 0u, p3 = 0u;
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const uint4 xa = sC[tid * 8 + ((2 * k) ^ (tid & 7))];
      const uint4 xb = sC[tid * 8 + ((2 * k + 1) ^ (tid & 7))];
      const uint32_t w[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
      uint32_t cur = 0u;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t code = (w[e >> 1] >> ((e & 1) * 16)) & 0xffffu;
        const uint32_t word = tbl[((code >> 4) << 5) + lane];
        cur |= ((word >> ((code & 15u) * 2u)) & 3u) << (2 * e);
      }
      const int tb = t0 + 16 * k;
      if (tb < c0 || tb + 16 > c1) cur &= span_mask(c0 - tb, c1 - tb);
      p0 = p1;
      p1 = p2;
      p2 = p3;
      p3 = cur;
    }
    const uint32_t p[4] = {p0, p1, p2, p3};
    A2ATS_PHASE(g_sel_phase, 9);
    uint32_t pk = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w)
      pk += (uint32_t)__popc(p[w] & 0x55555555u) | ((uint32_t)__popc(p[w] & 0xaaaaaaaau) << 16);
    uint32_t incl = pk;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) S.wsum[warp] = incl;
    __syncthreads();
    A2ATS_PHASE(g_sel_phase, 10);
    if (ch + 1 < nchunk) prefetch_chunk(a, cp_local, cb + kCH, c1, sC);  // sC is free
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kNW; ++w) {
      const uint32_t v = S.wsum[w];
      pre += (w < warp) ? v : 0u;
      tot += v;
    }
    const uint32_t ex = pre + incl - pk;  // 16-bit fields: a chunk holds <= 32768 tokens
    uint32_t gb = run_gt + (ex & 0xffffu), eb = run_eq + (ex >> 16);
    uint32_t e0 = p[0], e1 = p[1], e2 = p[2], e3 = p[3];
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
      uint32_t q = e0;
      e0 = e1;
      e1 = e2;
      e2 = e3;
      while (q) {  // selected / tied tokens in increasing token order
        const int bit = __ffs(q) - 1, j = bit >> 1;
        q &= ~(3u << (2 * j));
        const int t = t0 + 16 * w + j;
        // (positions are < cap by construction; the bound only guards against a
        //  caller-supplied hist that is inconsistent with the codes)
        if ((bit & 1) == 0) {  // class 1: above v*
          const uint32_t pos = gb + min(eb, m);
          if (pos < cap) selp[pos] = t;
          ++gb;
        } else {  // class 2: tied at v*
          if (eb < m && gb + eb < cap) selp[gb + eb] = t;
          ++eb;
        }
      }
    }
    run_gt += tot & 0xffffu;
    run_eq += tot >> 16;
  }
  return run_gt + min(run_eq, m);
}

// append: the step's new token n_ctx - 1 (encoded by the prep kernel) joins the histogram,
// after this pair's counts were taken (end of the kernel, off the critical path)
template <typename CT>
__device__ __forceinline__ void append_hist(const SelArgs& a, int pair, const CT* cp_local) {
  const int lo = a.shard_begin, t = a.n_ctx - 1;
  if (a.append_hist && a.hist && threadIdx.x == 0 && t >= lo && t < lo + a.shard_len)
    a.hist[(size_t)pair * a.L + cp_local[t - lo]] += 1;
}

// Window logits of the pair (Eq. 11 local rows: u_j = (q R_{i-j}) . k_j, exact per-row
// rotation on FP32 cores, base-2 scaled) for its first n_wl window tokens, from step inputs
// only; the caller writes them to wlog for the attention.  NT threads (512 or 256): thread
// <-> (row, heads g0, g0 + NT/64, ...); scratch: cs [64][64] float2 (fp64 angle per row
// group, then fp64 rotations by -f_m), K rows [64][16 chunks] and q [8][128] fp32, 16-B
// chunks XOR-swizzled by row.  Same arithmetic as the prep kernel's window role.
template <int NT>
__device__ void window_logits(const SelArgs& a, int pair, uint8_t* scratch, float (&out_acc)[512 / NT]) {
  constexpr int kHS = 512 / NT;  // head slots per thread
  const int tid = threadIdx.x, nw = a.n_wl, G = a.G;
  const int Hkv = gridDim.x / a.B;  // (one CTA per pair)
  const int b = pair / Hkv, h = pair - b * Hkv;
  float4* csS = reinterpret_cast<float4*>(scratch);
  uint4* kS = reinterpret_cast<uint4*>(scratch + 32768);
  float* sQ = reinterpret_cast<float*>(scratch + 32768 + 16384);
  const uint8_t* kbase = reinterpret_cast<const uint8_t*>(a.kc) + (size_t)pair * a.n_max * 256;
  if (tid < 128) {
    const int g = tid >> 4, e0 = (tid & 15) * 8;
    uint4 xq = make_uint4(0, 0, 0, 0);
    if (g < G) xq = ld_nc_u4(a.q + ((size_t)b * a.Hq + h * G + g) * kD + e0);
    const uint32_t w[4] = {xq.x, xq.y, xq.z, xq.w};
    float4* d = reinterpret_cast<float4*>(sQ + g * kD + e0);
    d[0] = make_float4(bf_lo(w[0]) * a.scale_log2, bf_hi(w[0]) * a.scale_log2, bf_lo(w[1]) * a.scale_log2,
                       bf_hi(w[1]) * a.scale_log2);
    d[1] = make_float4(bf_lo(w[2]) * a.scale_log2, bf_hi(w[2]) * a.scale_log2, bf_lo(w[3]) * a.scale_log2,
                       bf_hi(w[3]) * a.scale_log2);
  }
  for (int k = tid; k < nw * 16; k += NT) {
    const int r = k >> 4, c = k & 15;
    kS[r * 16 + (c ^ (r & 7))] = ld_nc_u4(kbase + (size_t)(a.win_lo + r - a.shard_begin) * 256 + c * 16);
  }
  {
    constexpr int kRows = 64 * 64 / NT;          // rows per thread of the cs table
    const int m = tid & 63, j0 = (tid >> 6) * kRows;  // rows [j0, j0 + kRows) of pair m
    if (j0 < nw) {
      const double f = a.rt.inv_freq[m];
      double sn, cn, sf, cf;
      sincos((double)(a.n_ctx - 1 - (a.win_lo + j0)) * f, &sn, &cn);  // r = i - t, t = win_lo + row
      sincos(f, &sf, &cf);
      float2* cs2 = reinterpret_cast<float2*>(csS);
#pragma unroll 1
      for (int row = j0; row < min(j0 + kRows, nw); ++row) {
        cs2[row * 64 + (((m >> 1) ^ (row & 7)) << 1) + (m & 1)] = make_float2((float)cn, (float)sn);
        const double c2 = cn * cf + sn * sf, s2 = sn * cf - cn * sf;  // r -> r - 1
        cn = c2;
        sn = s2;
      }
    }
  }
  __syncthreads();
  const int row = tid & 63, g0 = tid >> 6;  // heads g0 + s * (NT / 64)
  float acc[kHS];
#pragma unroll
  for (int s2 = 0; s2 < kHS; ++s2) acc[s2] = 0.f;
  if (row < nw && g0 < G) {
#pragma unroll 1
    for (int mb = 0; mb < 8; ++mb) {  // m = 8 mb + i; pairs (m, m + 64)
      const uint4 k1 = kS[row * 16 + (mb ^ (row & 7))];
      const uint4 k2 = kS[row * 16 + ((mb + 8) ^ (row & 7))];
      const uint32_t w1[4] = {k1.x, k1.y, k1.z, k1.w}, w2[4] = {k2.x, k2.y, k2.z, k2.w};
      float4 t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = csS[row * 32 + ((mb * 4 + j) ^ (row & 7))];
#pragma unroll
      for (int s2 = 0; s2 < kHS; ++s2) {
        const int g = g0 + s2 * (NT / 64);
        if (g < G) {
          const float* qa = sQ + g * kD + mb * 8;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float ka = (e & 1) ? bf_hi(w1[e >> 1]) : bf_lo(w1[e >> 1]);
            const float kb = (e & 1) ? bf_hi(w2[e >> 1]) : bf_lo(w2[e >> 1]);
            const float cv = (e & 1) ? t[e >> 1].z : t[e >> 1].x, sv = (e & 1) ? t[e >> 1].w : t[e >> 1].y;
            const float q1 = qa[e], q2 = qa[e + kHalf];
            acc[s2] = fmaf(cv, fmaf(q1, ka, q2 * kb), fmaf(sv, fmaf(q1, kb, -q2 * ka), acc[s2]));
          }
        }
      }
    }
  }
#pragma unroll
  for (int s2 = 0; s2 < kHS; ++s2) out_acc[s2] = acc[s2];
}

// wlog rows of the pair (after the dependency wait: the previous step's attention reads them)
template <int NT>
__device__ __forceinline__ void store_window_logits(const SelArgs& a, int pair, const float (&acc)[512 / NT]) {
  const int tid = threadIdx.x, row = tid & 63;
  if (row < a.n_wl) {
#pragma unroll
    for (int s2 = 0; s2 < 512 / NT; ++s2)
      a.wlog[((size_t)pair * 64 + row) * 8 + (tid >> 6) + s2 * (NT / 64)] = acc[s2];  // heads >= G: 0
  }
}

// Long contexts (several code chunks per pair), single GPU.
//   kThresh (grid P): counts, v*, m -> pinfo; compact 2-bit class table -> tblg.
//   kScanC (grid P x nchunk): one 32768-token chunk; classify, publish the chunk's
//   (#above, #tied) with a release store, sum the pair's earlier chunks' counts, emit.  A CTA
//   takes its chunk from a ticket counter when it starts, so every chunk it waits for was
//   handed to a CTA that started earlier (resident or done): the wait terminates whatever the
//   block scheduling order.  The last CTA to finish re-zeroes the counters; the threshold
//   kernel re-arms the descriptors of the next call.
template <int MODE>
__device__ __forceinline__ void split_body(const SelArgs& a, SelShared& S, int* cnt, uint32_t* key, uint32_t* tbl,
                                           uint32_t* skey, int* scnt, uint4* sC) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (MODE == kThresh) {
    const int pair = blockIdx.x;
    const uint16_t* cp_local = a.codes + (size_t)pair * a.n_max;
    float wacc[1] = {0.f};
    if (a.wlog) window_logits<kNT>(a, pair, reinterpret_cast<uint8_t*>(scnt + kSurvCap), wacc);
    load_cnt(a, pair, cnt, cp_local);
    pdl_wait();  // agg comes from the LUT kernel
    pdl_trigger();
    if (a.wlog) store_window_logits<kNT>(a, pair, wacc);
    uint32_t kstar = 0, m = 0;
    if (a.keff > 0) {
      load_keys(a, S, pair, cnt, key);
      find_level(a, S, cnt, key, a.keff, skey, scnt);
      kstar = S.s_kstar;
      m = S.s_m;
      for (int w = tid; w < a.W; w += kNT) {  // compact class table: 16 codewords x 2 bits per word
        uint32_t x = 0;
#pragma unroll 1
        for (int e = 0; e < 16 && w * 16 + e < a.L; ++e) {
          const uint32_t k = key[w * 16 + e];
          x |= ((k < kstar) ? 1u : ((k == kstar) ? 2u : 0u)) << (2 * e);
        }
        a.tblg[(size_t)pair * a.W + w] = x;
      }
    }
    if (tid == 0) {
      a.pinfo[pair * 4 + 0] = kstar;
      a.pinfo[pair * 4 + 1] = m;
      a.pinfo[pair * 4 + 2] = (uint32_t)a.keff;
    }
    // re-arm the pair's chunk descriptors (the previous call's scan is complete: this runs
    // after the dependency wait, and the scan kernel of this call waits for this one)
    for (int c = tid; c < a.desc_stride; c += kNT) a.desc[(size_t)pair * a.desc_stride + c] = 0ull;
    append_hist(a, pair, cp_local);
    return;
  }
  // kScanC
  __shared__ int s_item;
  if (tid == 0) s_item = (int)atomicAdd(a.tickets, 1u);  // chunk item in start order
  __syncthreads();
  auto finish = [&]() {  // the last CTA out leaves the counters zero for the next call
    if (tid == 0 && atomicAdd(a.tickets + 1, 1u) == gridDim.x - 1) {
      a.tickets[0] = 0u;
      a.tickets[1] = 0u;
    }
  };
  const int pair = s_item / a.nchunk, ch = s_item - pair * a.nchunk;
  const uint16_t* cp_local = a.codes + (size_t)pair * a.n_max;
  const int c0 = a.c0, c1 = a.c1;
  const int cb = ((c0 >> 3) << 3) + ch * kCH;
  if (cb < c1) prefetch_chunk(a, cp_local, cb, c1, sC);
  pdl_wait();  // pinfo / tblg come from kThresh
  pdl_trigger();
  const uint32_t kstar = __ldcg(a.pinfo + pair * 4 + 0), m = __ldcg(a.pinfo + pair * 4 + 1);
  const uint32_t cap = __ldcg(a.pinfo + pair * 4 + 2);
  if (cap == 0 || cb >= c1) {
    cp_async_wait<0>();
    finish();
    return;
  }
  for (int it = tid; it < a.W * 2; it += kNT) {  // class table, replicated 32x (2 threads per word)
    const int w = it >> 1;
    const uint32_t x = __ldcg(a.tblg + (size_t)pair * a.W + w);
    uint4* dst = reinterpret_cast<uint4*>(tbl + w * 32 + (it & 1) * 16);
    const uint4 v = make_uint4(x, x, x, x);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[(q + w) & 3] = v;
  }
  cp_async_wait<0>();
  __syncthreads();
  A2ATS_TL(g_selc_tl, 2);
  const int t0 = cb + tid * kTPT;
  uint32_t p0 = 0u, p1 = 0u, p2 = 0u, p3 = 0u;
#pragma unroll 1
  for (int k = 0; k < 4; ++k) {
    const uint4 xa = sC[tid * 8 + ((2 * k) ^ (tid & 7))];
    const uint4 xb = sC[tid * 8 + ((2 * k + 1) ^ (tid & 7))];
    const uint32_t w8[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    uint32_t cur = 0u;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const uint32_t code = (w8[e >> 1] >> ((e & 1) * 16)) & 0xffffu;
      const uint32_t word = tbl[((code >> 4) << 5) + lane];
      cur |= ((word >> ((code & 15u) * 2u)) & 3u) << (2 * e);
    }
    const int tb = t0 + 16 * k;
    if (tb < c0 || tb + 16 > c1) cur &= span_mask(c0 - tb, c1 - tb);
    p0 = p1;
    p1 = p2;
    p2 = p3;
    p3 = cur;
  }
  uint32_t pk = (uint32_t)__popc(p0 & 0x55555555u) + (uint32_t)__popc(p1 & 0x55555555u) +
                (uint32_t)__popc(p2 & 0x55555555u) + (uint32_t)__popc(p3 & 0x55555555u);
  pk |= ((uint32_t)__popc(p0 & 0xaaaaaaaau) + (uint32_t)__popc(p1 & 0xaaaaaaaau) +
         (uint32_t)__popc(p2 & 0xaaaaaaaau) + (uint32_t)__popc(p3 & 0xaaaaaaaau)) << 16;
  uint32_t incl = pk;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) S.wsum[warp] = incl;
  __syncthreads();
  A2ATS_TL(g_selc_tl, 3);
  uint32_t pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kNW; ++w) {
    const uint32_t v = S.wsum[w];
    pre += (w < warp) ? v : 0u;
    tot += v;
  }
  unsigned long long* desc = a.desc + (size_t)pair * a.desc_stride;
  if (warp == 0) {  // publish this chunk's counts, then sum the earlier chunks' (one lane each)
    if (lane == 0)
      st_release_u64(desc + ch, (1ull << 63) | ((unsigned long long)(tot >> 16) << 31) | (tot & 0xffffu));
    uint32_t gb = 0, eb = 0;
#pragma unroll 1
    for (int c = lane; c < ch; c += 32) {
      unsigned long long v;
      while (!((v = ld_acquire_u64(desc + c)) >> 63)) __nanosleep(32);
      gb += (uint32_t)(v & 0x7fffffffull);
      eb += (uint32_t)((v >> 31) & 0x7fffffffull);
    }
    gb = __reduce_add_sync(0xffffffffu, gb);
    eb = __reduce_add_sync(0xffffffffu, eb);
    if (lane == 0) {
      S.s_before[0] = gb;
      S.s_before[1] = eb;
    }
  }
  __syncthreads();
  A2ATS_TL(g_selc_tl, 4);
  const uint32_t ex = pre + incl - pk;
  uint32_t gb = S.s_before[0] + (ex & 0xffffu), eb = S.s_before[1] + (ex >> 16);
  int32_t* selp = a.sel + (size_t)pair * a.sel_stride;
  uint32_t e0 = p0, e1 = p1, e2 = p2, e3 = p3;
#pragma unroll 1
  for (int w = 0; w < 4; ++w) {
    uint32_t q = e0;
    e0 = e1;
    e1 = e2;
    e2 = e3;
    while (q) {  // selected / tied tokens in increasing token order
      const int bit = __ffs(q) - 1, j = bit >> 1;
      q &= ~(3u << (2 * j));
      const int t = t0 + 16 * w + j;
      if ((bit & 1) == 0) {
        const uint32_t pos = gb + min(eb, m);
        if (pos < cap) selp[pos] = t;
        ++gb;
      } else {
        if (eb < m && gb + eb < cap) selp[gb + eb] = t;
        ++eb;
      }
    }
  }
  finish();
}

// ---------------------------------------------------------------- emission helper
// emit the tokens of a 16-token class word: above-v* fields at base++, tied fields (rare)
// through the quota; returns nothing, advances gb / eb
__device__ __forceinline__ void emit16(uint32_t q, int t0, uint32_t& gb, uint32_t& eb, uint32_t m, uint32_t cap,
                                       int32_t* selp) {
  if ((q & 0xaaaaaaaau) == 0u) {  // no tied token: positions gb + min(eb, m) .. + n - 1
    const uint32_t n = __popc(q), pos = gb + min(eb, m);
    gb += n;
    if (pos + n <= cap) {  // (always, unless hist is inconsistent with the codes)
      int32_t* dst = selp + pos + n;
      do {  // highest token first
        const int bit = 31 - __clz(q);
        q ^= 1u << bit;
        *--dst = t0 + (bit >> 1);
      } while (q);
    }
    return;
  }
  while (q) {  // in increasing token order
    const int bit = __ffs(q) - 1;
    q &= q - 1u;
    const int t = t0 + (bit >> 1);
    if ((bit & 1) == 0) {  // above v*
      const uint32_t pos = gb + min(eb, m);
      if (pos < cap) selp[pos] = t;
      ++gb;
    } else {  // tied at v*: the first m in token order
      if (eb < m && gb + eb < cap) selp[gb + eb] = t;
      ++eb;
    }
  }
}

// ---------------------------------------------------------------- long contexts with hist
// Two kernels after the LUT (prep) kernel:
//  select_thresh_kernel (grid P, 256 threads, four resident per SM: one wave at C4): per
//    pair, the window rows' logits (for the attention) and the counts (hist - sink/window
//    codes) before the dependency wait, then keys, v*, m,
//    E = #{candidates at level v*}, and the compact 2-bit class table -> tblg, (v*, m, K_eff,
//    E) -> pinfo; appends the step's new token to hist.
//  select_scan_kernel: a persistent grid (one 1024-thread CTA per SM) over 2P work units:
//    unit u < P streams the first half of pair u's candidate stages FORWARD, unit u >= P the
//    second half of pair u - P BACKWARD.  The halves exchange nothing: with D = E - m, the
//    forward half keeps its first m tied tokens and writes ascending from position 0; the
//    backward half drops the last D tied tokens it meets and writes descending from
//    position K_eff - 1 (together: exactly the first m ties in token order, the lowest-index
//    tie-break of reading Q12).  2P units over the SMs balance to within one half-pair.
//    Codes arrive through a ring of 32-KB stages (one TMA box of 256 128-B rows each,
//    SWIZZLE_128B, mbarrier completion) that runs ahead across unit boundaries and is
//    issued before the dependency wait (codes are step inputs).  Each pair's class table
//    is replicated 32x in shared memory (lane l reads replica l: conflict-free gather by
//    code), double-buffered: the next unit's table is written during the current one.
constexpr int kPAll = 1024;          // scan kernel threads
constexpr int kPRound = 256 * 64;    // tokens per stage: one TMA box of 256 128-B rows (32 KB)
#ifndef A2ATS_SCAN_STAGES
#define A2ATS_SCAN_STAGES 5
#endif
constexpr int kPStage = A2ATS_SCAN_STAGES;  // ring stages (32 KB each): 5 fit beside one class table
constexpr int kTT = 256;             // threshold kernel threads
constexpr int kTSurv = 1024;         // its survivor list capacity

struct PipeUnit {
  uint32_t m, D, cap, pad;
};


__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
// classify8 with the lane's table replica at shared address tl = table | 4 * lane, the
// table 32-KB aligned in the shared window and codes < 4096: word (code >> 4) of the replica
// is at tl | (code >> 4) << 7, one LOP3 per code (no add)
__device__ __forceinline__ uint32_t classify8s(uint32_t tl, uint4 v) {
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


// backward emission of a 16-token class word: tokens in decreasing order; a token with
// ga above-v* and ea tied tokens after it (in this unit) goes to top - 1 - (ga + max(ea - D, 0));
// a tied token is kept iff ea >= D
__device__ __forceinline__ void emit16_rev(uint32_t q, int t0, uint32_t& ga, uint32_t& ea, uint32_t D, uint32_t top,
                                           int32_t* selp) {
  if ((q & 0xaaaaaaaau) == 0u) {
    const uint32_t n = __popc(q), used = ga + (ea > D ? ea - D : 0u);
    ga += n;
    if (used + n <= top) {
      int32_t* dst = selp + (top - used - n);
      do {  // lowest token first, ascending positions
        const int bit = __ffs(q) - 1;
        q &= q - 1u;
        *dst++ = t0 + (bit >> 1);
      } while (q);
    }
    return;
  }
  while (q) {
    const int bit = 31 - __clz(q);
    q ^= 1u << bit;
    const int t = t0 + (bit >> 1);
    if ((bit & 1) == 0) {
      const uint32_t used = ga + (ea > D ? ea - D : 0u);
      if (used < top) selp[top - 1 - used] = t;
      ++ga;
    } else {
      if (ea >= D) {
        const uint32_t used = ga + ea - D;
        if (used < top) selp[top - 1 - used] = t;
      }
      ++ea;
    }
  }
}

struct PipeGeom {
  int first, R, R0, c1al;
};
__device__ __forceinline__ PipeGeom pipe_geom(const SelArgs& a) {
  PipeGeom g;
  g.first = (a.c0 >> 6) << 6;
  g.c1al = (a.c1 + 7) & ~7;
  g.R = (a.c1 - g.first + kPRound - 1) / kPRound;
  g.R0 = (g.R + 1) >> 1;
  return g;
}

// Thresholds with register-resident codewords: thread t holds the keys and candidate counts
// of codewords [PT t, PT t + PT) (L <= PT * NT): the range, the 256-bin weighted value
// histogram, the survivors of the K-th bin (one block scan), their ranking (or byte passes
// over the registers when there are more than NT), without re-reading shared memory.  Same
// selection rule and bins as find_level.
template <int PT>
__device__ __forceinline__ void load_c_regs(const SelArgs& a, const int* cnt, int (&c)[PT]) {
  const int l0 = threadIdx.x * PT;
#pragma unroll
  for (int q = 0; q < PT / 4; ++q) {
    int4 v = make_int4(0, 0, 0, 0);
    if (l0 + 4 * q + 4 <= a.L) {
      v = *reinterpret_cast<const int4*>(cnt + l0 + 4 * q);
    } else {
      v.x = (l0 + 4 * q + 0 < a.L) ? cnt[l0 + 4 * q + 0] : 0;
      v.y = (l0 + 4 * q + 1 < a.L) ? cnt[l0 + 4 * q + 1] : 0;
      v.z = (l0 + 4 * q + 2 < a.L) ? cnt[l0 + 4 * q + 2] : 0;
      v.w = (l0 + 4 * q + 3 < a.L) ? cnt[l0 + 4 * q + 3] : 0;
    }
    c[4 * q] = v.x;
    c[4 * q + 1] = v.y;
    c[4 * q + 2] = v.z;
    c[4 * q + 3] = v.w;
  }
}

// PRE: the caller set S.s_kmin = ~0, S.s_kmax = 0 and zeroed S.bins before a barrier (saves one)
template <int NT, int PT, bool PRE = false>
__device__ __forceinline__ void level_regs(const SelArgs& a, SelShared& S, int pair, const int (&c)[PT],
                                           uint32_t (&k)[PT], uint32_t* skey, int* scnt, int survcap,
                                           uint32_t& kstar_out, uint32_t& m_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, l0 = tid * PT;
  {
    const float* aggp = a.agg + (size_t)pair * a.L + l0;
    float f[PT];
#pragma unroll
    for (int q = 0; q < PT / 4; ++q) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (l0 + 4 * q + 4 <= a.L) {
        v = __ldcg(reinterpret_cast<const float4*>(aggp + 4 * q));
      } else {
        v.x = (l0 + 4 * q + 0 < a.L) ? __ldcg(aggp + 4 * q + 0) : 0.f;
        v.y = (l0 + 4 * q + 1 < a.L) ? __ldcg(aggp + 4 * q + 1) : 0.f;
        v.z = (l0 + 4 * q + 2 < a.L) ? __ldcg(aggp + 4 * q + 2) : 0.f;
        v.w = (l0 + 4 * q + 3 < a.L) ? __ldcg(aggp + 4 * q + 3) : 0.f;
      }
      f[4 * q] = v.x;
      f[4 * q + 1] = v.y;
      f[4 * q + 2] = v.z;
      f[4 * q + 3] = v.w;
    }
    uint32_t kmn = 0xffffffffu, kmx = 0u;
#pragma unroll
    for (int e = 0; e < PT; ++e) {
      k[e] = ~ordered_key(f[e]);
      if (c[e] > 0) {
        kmn = min(kmn, k[e]);
        kmx = max(kmx, k[e]);
      }
    }
    kmn = __reduce_min_sync(0xffffffffu, kmn);
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    if (!PRE) {
      if (tid == 0) {
        S.s_kmin = 0xffffffffu;
        S.s_kmax = 0u;
      }
      for (int i = tid; i < 256; i += NT) S.bins[i] = 0;
      __syncthreads();
    }
    if (lane == 0) {
      atomicMin(&S.s_kmin, kmn);
      atomicMax(&S.s_kmax, kmx);
    }
    __syncthreads();
  }
  if (NT == 256 && tid == 0) A2ATS_TLX(g_sel_tl, 5);
  const int keff = a.keff;
  const uint32_t kmn = S.s_kmin, kmx = S.s_kmax;
  if (kmn == kmx) {  // a single level holds every candidate
    kstar_out = kmn;
    m_out = (uint32_t)keff;
    return;
  }
  // 256 bins over the candidates' VALUE range (the key range spans the sign boundary of the
  // floats: binning keys by shifts puts most candidates into a few bins -- measured 8x the rank)
  auto key_val = [](uint32_t kk) {
    const uint32_t o = ~kk;
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
  };
  const float amax = key_val(kmn), amin = key_val(kmx);
  const float scale = 255.99f / (amax - amin);
  uint32_t binp[PT / 4];  // PT bins, one byte each
#pragma unroll
  for (int q = 0; q < PT / 4; ++q) binp[q] = 0u;
#pragma unroll
  for (int e = 0; e < PT; ++e) {
    const float d = amax - key_val(k[e]);
    const uint32_t b = d > 0.f ? (uint32_t)min(255, (int)(d * scale)) : 0u;
    binp[e >> 2] |= b << (8 * (e & 3));
    if (c[e] > 0) atomicAdd(&S.bins[b], c[e]);
  }
  auto bin = [&](int e) { return (binp[e >> 2] >> (8 * (e & 3))) & 255u; };
  __syncthreads();
  if (warp == 0) pick_digit(S, keff);
  __syncthreads();
  if (NT == 256 && tid == 0) A2ATS_TLX(g_sel_tl, 6);
  const uint32_t bstar = (uint32_t)S.s_digit;
  int kk = S.s_kk;
  uint32_t kmask = 0u;
#pragma unroll
  for (int e = 0; e < PT; ++e)
    if (c[e] > 0 && bin(e) == bstar) kmask |= 1u << e;
  const int nk = __popc(kmask);
  int incl = nk;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) S.wsum[warp] = (uint32_t)incl;
  __syncthreads();
  int base = incl - nk, nsurv = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    const int v = (int)S.wsum[w];
    base += (w < warp) ? v : 0;
    nsurv += v;
  }
  if (nsurv <= NT && nsurv <= survcap) {
#pragma unroll
    for (int e = 0; e < PT; ++e)
      if ((kmask >> e) & 1u) {
        skey[base] = k[e];
        scnt[base] = c[e];
        ++base;
      }
  }
  __syncthreads();
  if (NT == 256 && tid == 0) A2ATS_TLX(g_sel_tl, 7);
  if (nsurv <= NT && nsurv <= survcap) {  // rank each survivor directly: #(< v*) < kk <= #(<= v*)
    if (tid < nsurv) {
      const uint32_t ki = skey[tid];
      int less = 0, leq = 0;
#pragma unroll 4
      for (int jj = 0; jj < nsurv; ++jj) {
        const uint32_t kj = skey[jj];
        const int cj = scnt[jj];
        less += (kj < ki) ? cj : 0;
        leq += (kj <= ki) ? cj : 0;
      }
      if (less < kk && kk <= leq) {
        S.s_kstar = ki;
        S.s_m = (uint32_t)(kk - less);
      }
    }
  } else {  // many survivors: byte passes over the registers, restricted to bin b*
    uint32_t prefix = 0, mask = 0;
    for (int pass = 3; pass >= 0; --pass) {
      const int shift = 8 * pass;
      for (int i = tid; i < 256; i += NT) S.bins[i] = 0;
      __syncthreads();
#pragma unroll
      for (int e = 0; e < PT; ++e)
        if (c[e] > 0 && bin(e) == bstar && (k[e] & mask) == prefix) atomicAdd(&S.bins[(k[e] >> shift) & 255u], c[e]);
      __syncthreads();
      if (warp == 0) pick_digit(S, kk);
      __syncthreads();
      prefix |= (uint32_t)S.s_digit << shift;
      mask |= 0xffu << shift;
      kk = S.s_kk;
    }
    if (tid == 0) {
      S.s_kstar = prefix;
      S.s_m = (uint32_t)kk;
    }
  }
  __syncthreads();
  kstar_out = S.s_kstar;
  m_out = S.s_m;
}

// 2-bit classes of the thread's PT codewords (codeword e at bits 2e) and their candidates at v*
template <int PT>
__device__ __forceinline__ uint32_t class_bits(const uint32_t (&k)[PT], const int (&c)[PT], uint32_t kstar, int& e_cnt) {
  uint32_t x = 0;
#pragma unroll
  for (int e = 0; e < PT; ++e) {
    x |= ((k[e] < kstar) ? 1u : ((k[e] == kstar) ? 2u : 0u)) << (2 * e);
    if (k[e] == kstar) e_cnt += max(c[e], 0);
  }
  return x;
}

__global__ __launch_bounds__(kTT, 4) void select_thresh_kernel(SelArgs a) {
  A2ATS_TL(g_sel_tl, 0);
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ SelShared S;
  const int tid = threadIdx.x, lane = tid & 31, pair = blockIdx.x;
  const int L4 = (a.L + 3) & ~3;
  int* cnt = reinterpret_cast<int*>(sm);
  uint32_t* skey = sm + L4;
  int* scnt = reinterpret_cast<int*>(skey + kTSurv);
  const uint16_t* cp = a.codes + (size_t)pair * a.n_max;
  float wacc[512 / kTT];
  if (a.wlog) {  // the pair's window-row logits (step inputs only; scratch aliases cnt / survivors)
    window_logits<kTT>(a, pair, reinterpret_cast<uint8_t*>(sm), wacc);
    __syncthreads();
  }
  load_cnt<kTT>(a, pair, cnt, cp);  // step inputs
  int c[16];
  load_c_regs<16>(a, cnt, c);
  pdl_wait();                       // agg comes from the prep kernel
  pdl_trigger();
  A2ATS_TL(g_sel_tl, 3);
  if (a.wlog) store_window_logits<kTT>(a, pair, wacc);  // the previous step's attention has read wlog
  append_hist(a, pair, cp);         // counts taken: the new token joins hist
  if (tid == 0) S.s_eq = 0;
  uint32_t k[16], kstar, m;
  level_regs<kTT, 16>(a, S, pair, c, k, skey, scnt, kTSurv, kstar, m);
  A2ATS_TL(g_sel_tl, 4);
  // this thread's 16 codewords = word tid of the compact class table; E = #candidates at v*
  int e_cnt = 0;
  const uint32_t x = class_bits<16>(k, c, kstar, e_cnt);
  if (tid < a.W) a.tblg[(size_t)pair * a.W + tid] = x;
  e_cnt = __reduce_add_sync(0xffffffffu, e_cnt);
  if (lane == 0 && e_cnt) atomicAdd(&S.s_eq, e_cnt);
  __syncthreads();
  if (tid == 0) {
    a.pinfo[pair * 4 + 0] = kstar;
    a.pinfo[pair * 4 + 1] = m;
    a.pinfo[pair * 4 + 2] = (uint32_t)a.keff;
    a.pinfo[pair * 4 + 3] = (uint32_t)S.s_eq;
  }
  A2ATS_TL(g_sel_tl, 1);
}

// ---------------------------------------------------------------- sharded step, replicated histograms
// Collective-free exact global top-K: every rank holds the global code histogram
// and every rank's histogram of tokens [0, n-1), plus the codes of the sinks and of the latest
// WR tokens (the caller-visible shard state, updated identically on every rank from the step's
// all-gather).  So every rank derives the same K-th level v* and tie quota m (the LUT is
// bitwise identical on every rank), and its own share of the ties -- the first m tied tokens in
// global order go to the lowest ranks first (reading Q12) -- without exchanging anything:
//   cand_r[l] = hist_r[r][l] - #(rank r's sink / window tokens < n-1 with code l)
//   E_before  = sum over ranks r' < rank of cand_r'[l] for the tied codes l (agg_l == v*)
//   m_local   = clamp(m - E_before, 0, E_local),  K_eff_local = #above_local + m_local.
// (v*, m_local, K_eff_local, E_local) and the class table feed the persistent scan over the
// rank's local candidate range, exactly as on one GPU.  The owner of the new token n-1 also
// copies its code (just encoded by the prep kernel) into the all-gather message.
__device__ __forceinline__ int owner_of(const SelArgs& a, int t) {
  int r = 0;
  while (r + 1 < a.world && t >= a.bounds[r + 1]) ++r;
  return r;
}

__global__ __launch_bounds__(kTT, 4) void select_shard_thresh_kernel(SelArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ SelShared S;
  __shared__ int s_above, s_eq, s_before;
  const int tid = threadIdx.x, lane = tid & 31, pair = blockIdx.x;
  const int L4 = (a.L + 3) & ~3;
  int* cnt = reinterpret_cast<int*>(sm);        // [L] global candidate counts (registers after load_c_regs)
  int* cnl = cnt + L4;                          // [L] this rank's candidate counts
  uint32_t* keys = reinterpret_cast<uint32_t*>(cnt);  // [L] keys, once cnt is dead
  uint32_t* skey = reinterpret_cast<uint32_t*>(cnl + L4);
  int* scnt = reinterpret_cast<int*>(skey + kTSurv);
  const size_t PL = (size_t)gridDim.x * a.L;
  float wacc[512 / kTT];
  if (a.wlog) {  // this rank's window-row logits (step inputs only; scratch aliases the counts)
    window_logits<kTT>(a, pair, reinterpret_cast<uint8_t*>(sm), wacc);
    __syncthreads();
  }
  // step inputs (replicated state): counts of tokens [0, n-1) minus sinks and window tokens
  for (int l = tid; l < a.L; l += kTT) {
    cnt[l] = a.hist_g[(size_t)pair * a.L + l];
    cnl[l] = a.hist_r[(size_t)a.rank * PL + (size_t)pair * a.L + l];
  }
  if (tid == 0) s_above = s_eq = s_before = 0;
  __syncthreads();
  const int n = a.n_ctx, t_new = n - 1;
  const int n_stat = a.n_s + (t_new - a.w0);  // sinks + window tokens other than the new one
  for (int i = tid; i < n_stat; i += kTT) {
    const int t = i < a.n_s ? i : a.w0 + (i - a.n_s);
    const int code = i < a.n_s ? a.sinkc[(size_t)pair * a.n_sink_cap + t] : a.ring[(size_t)pair * a.WR + (t % a.WR)];
    atomicSub(&cnt[code], 1);
    if (owner_of(a, t) == a.rank) atomicSub(&cnl[code], 1);
  }
  __syncthreads();
  int c[16];
  load_c_regs<16>(a, cnt, c);
  __syncthreads();  // cnt is dead: its space holds the keys below
  pdl_wait();  // agg from the prep kernel (and the new token's code from its encode role)
  pdl_trigger();
  if (a.wlog) store_window_logits<kTT>(a, pair, wacc);  // the previous step's attention has read wlog
  if (a.send_codes && a.rank == a.owner && tid == 0)
    a.send_codes[pair] = a.codes[(size_t)pair * a.n_max + (t_new - a.shard_begin)];
  uint32_t k[16], kstar = 0u, m = 0u;
  if (a.keff > 0) {
    level_regs<kTT, 16>(a, S, pair, c, k, skey, scnt, kTSurv, kstar, m);
  } else {
    const float* aggp = a.agg + (size_t)pair * a.L;
#pragma unroll
    for (int e = 0; e < 16; ++e) k[e] = tid * 16 + e < a.L ? ~ordered_key(__ldcg(aggp + tid * 16 + e)) : 0u;
    kstar = 0u;  // no key is below 0: nothing above; ties (key 0) are not candidates
  }
  // the compact class table (this thread's 16 codewords = word tid) and the keys into smem
  uint32_t x = 0u;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int l = tid * 16 + e;
    if (l < a.L) keys[l] = k[e];
    if (a.keff > 0) x |= ((k[e] < kstar) ? 1u : ((k[e] == kstar) ? 2u : 0u)) << (2 * e);
  }
  __syncthreads();
  // this rank's counts above / at v* and the lower ranks' ties at v*
  int above = 0, eq = 0, before = 0;
  if (a.keff > 0) {
    for (int l = tid; l < a.L; l += kTT) {
      const uint32_t kl = keys[l];
      if (kl < kstar) {
        above += cnl[l];
      } else if (kl == kstar) {
        eq += cnl[l];
        for (int r = 0; r < a.rank; ++r) before += a.hist_r[(size_t)r * PL + (size_t)pair * a.L + l];
      }
    }
  }
  if (tid < a.W) a.tblg[(size_t)pair * a.W + tid] = x;
  above = __reduce_add_sync(0xffffffffu, above);
  eq = __reduce_add_sync(0xffffffffu, eq);
  before = __reduce_add_sync(0xffffffffu, before);
  if (lane == 0) {
    atomicAdd(&s_above, above);
    atomicAdd(&s_eq, eq);
    atomicAdd(&s_before, before);
  }
  __syncthreads();
  // lower ranks' sink / window tokens at v* are in their histograms but are not candidates
  if (a.keff > 0) {
    for (int i = tid; i < n_stat; i += kTT) {
      const int t = i < a.n_s ? i : a.w0 + (i - a.n_s);
      const int code = i < a.n_s ? a.sinkc[(size_t)pair * a.n_sink_cap + t] : a.ring[(size_t)pair * a.WR + (t % a.WR)];
      if (keys[code] == kstar && owner_of(a, t) < a.rank) atomicSub(&s_before, 1);
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int e_loc = s_eq;
    const int m_loc = a.keff > 0 ? min(max((int)m - s_before, 0), e_loc) : 0;
    const int cap = a.keff > 0 ? s_above + m_loc : 0;
    a.pinfo[pair * 4 + 0] = kstar;
    a.pinfo[pair * 4 + 1] = (uint32_t)m_loc;
    a.pinfo[pair * 4 + 2] = (uint32_t)cap;
    a.pinfo[pair * 4 + 3] = (uint32_t)e_loc;
    a.nsel_out[pair] = cap;
  }
}

// Stream one unit (half of a pair's candidate stages).  Super-rounds of two stages (32768
// tokens): thread t takes stage t >> 9, row (t & 511) >> 1 (64 tokens), half t & 1 (32
// consecutive tokens, pieces 4 (t & 1) .. + 3, read through the SWIZZLE_128B layout:
// conflict-free); one warp scan + one CTA barrier per super-round give the output offsets,
// then the two freed stages are refilled.  At the end of the unit the next unit's table is
// written into the other buffer (its loads were issued at unit start; the previous unit,
// which read that buffer, finished before this one began).
struct ScanCtx {
  const SelArgs& a;
  const PipeGeom& g;
  uint32_t ring, tbl0;  // shared addresses
  uint64_t* full;
  uint32_t* sTot;       // [2][32]
  int nchunks;
};

template <bool FWD, class Issue, class Expand>
__device__ __forceinline__ void scan_unit(const ScanCtx& c, int buf, int pair, int nr, const PipeUnit pu, int& j,
                                          Issue& issue, Expand& expand) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t tl = (c.tbl0 + buf * 32768u) | ((uint32_t)lane * 4u);
  const int half = tid >> 9;  // 0: lower stage of the super-round, 1: upper
  const int row = (tid & 511) >> 1, hp = tid & 1;
  int32_t* selp = c.a.sel + (size_t)pair * c.a.sel_stride;
  uint32_t run_gt = 0, run_eq = 0;
#pragma unroll 1
  for (int i = 0; i < nr; i += 2) {
    const bool two = i + 1 < nr;
    // stages of this super-round: forward i (lower), i + 1 (upper); backward i (upper), i + 1 (lower)
    const int r_lo = FWD ? i : c.g.R - 2 - i;  // round index of the lower stage (may be absent)
    const bool mine = FWD ? (half == 0 || two) : (half == 1 || two);
    const int jmine = FWD ? j + half : j + (1 - half);
    const int tr = c.g.first + (r_lo + half) * kPRound, t0 = tr + row * 64 + hp * 32;
    uint4 v[4];
    if (mine) {
      const int s = jmine % kPStage;
      umma::mbar_wait(&c.full[s], (uint32_t)(jmine / kPStage) & 1u);
      const uint32_t st = c.ring + s * (kPRound * 2) + row * 128;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = lds_v4(st + (((4 * hp + q) ^ (row & 7)) << 4));
      const int npiece = (min(tr + kPRound, c.g.c1al) - tr) >> 3;
      if (npiece < kPRound / 8) {  // last stage: codes past the range may be past n_ctx (undefined)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (row * 8 + 4 * hp + q >= npiece) v[q] = make_uint4(0, 0, 0, 0);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = make_uint4(0, 0, 0, 0);
    }
    uint32_t cw[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) cw[q] = classify8s(tl, v[2 * q]) | (classify8s(tl, v[2 * q + 1]) << 16);
    if (!mine) {
      cw[0] = cw[1] = 0u;
    } else if (t0 < c.a.c0 || t0 + 32 > c.a.c1) {  // tokens outside [c0, c1)
#pragma unroll
      for (int q = 0; q < 2; ++q) cw[q] &= span_mask(c.a.c0 - t0 - 16 * q, c.a.c1 - t0 - 16 * q);
    }
    const uint32_t pk = (uint32_t)(__popc(cw[0] & 0x55555555u) + __popc(cw[1] & 0x55555555u)) |
                        ((uint32_t)(__popc(cw[0] & 0xaaaaaaaau) + __popc(cw[1] & 0xaaaaaaaau)) << 16);
    uint32_t incl = pk;  // 16-bit fields: 32768 tokens per super-round
    if (FWD) {
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
    } else {
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, incl, off);
        if (lane + off < 32) incl += y;
      }
    }
    const int par = (i >> 1) & 1;
    if (lane == (FWD ? 31 : 0)) c.sTot[par * 32 + warp] = incl;
    if (tid == 0 && j < 2) A2ATS_TLX(g_selc_tl, 5);
    __syncthreads();  // every thread has read its stage (and the previous unit is done with the other table)
    if (tid == 0 && j < 2) A2ATS_TLX(g_selc_tl, 6);
    if (tid == 0) {
      if (j + kPStage < c.nchunks) issue(j + kPStage);
      if (two && j + 1 + kPStage < c.nchunks) issue(j + 1 + kPStage);
    }
    j += two ? 2 : 1;
    // lane w holds warp w's total: the super-round total and this warp's offset
    const uint32_t wv = c.sTot[par * 32 + lane];
    const uint32_t tot = __reduce_add_sync(0xffffffffu, wv);
    const uint32_t pre = __reduce_add_sync(0xffffffffu, (FWD ? (lane < warp) : (lane > warp)) ? wv : 0u);
    const uint32_t ex = pre + incl - pk;
    uint32_t gb = run_gt + (ex & 0xffffu), eb = run_eq + (ex >> 16);
    if (pk) {
      const int te = t0 + c.a.sel_base;  // emitted index (sharded step: local -> global)
      if (FWD) {
        if (cw[0]) emit16(cw[0], te, gb, eb, pu.m, pu.cap, selp);
        if (cw[1]) emit16(cw[1], te + 16, gb, eb, pu.m, pu.cap, selp);
      } else {
        if (cw[1]) emit16_rev(cw[1], te + 16, gb, eb, pu.D, pu.cap, selp);
        if (cw[0]) emit16_rev(cw[0], te, gb, eb, pu.D, pu.cap, selp);
      }
    }
    run_gt += tot & 0xffffu;
    run_eq += tot >> 16;
    if (tid == 0 && j <= 2) A2ATS_TLX(g_selc_tl, 7);
  }
  expand();  // the next unit's table into the other buffer (its loads were issued at unit start)
}

__global__ __launch_bounds__(kPAll, 1) void select_scan_kernel(const __grid_constant__ CUtensorMap tmK, SelArgs a) {
  A2ATS_TL(g_selc_tl, 0);
  extern __shared__ __align__(128) uint8_t smp[];
  __shared__ __align__(16) uint32_t sTot[2][32];
  __shared__ __align__(8) uint64_t full[kPStage];
  const int P = a.P, nblk = gridDim.x, W = a.W;
  const int tid = threadIdx.x;
  // tables at the first 32-KB boundary of the shared window ([2][32 KB], 32x-replicated class
  // words: OR-addressing in classify8s), then the ring ([kPStage][32 KB], 1024-B aligned).  One
  // table buffer: the next unit's table is written by expand() after the unit's last super-round
  // barrier, which every warp passes only once it has classified its last tokens of the unit
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smp);
  const uint32_t tsh = (sbase + 32767u) & ~32767u;
  uint32_t* tbl0 = reinterpret_cast<uint32_t*>(smp + (tsh - sbase));
  uint8_t* ring = smp + (tsh - sbase) + 32768;
  const PipeGeom g = pipe_geom(a);
  const int R1 = g.R - g.R0;
  const int nunit = (2 * P - (int)blockIdx.x + nblk - 1) / nblk;        // units u = blockIdx.x + k * nblk
  const int nk0 = max(0, min(nunit, (P - (int)blockIdx.x + nblk - 1) / nblk));  // forward ones (u < P)
  const int nchunks = nk0 * g.R0 + (nunit - nk0) * R1;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < kPStage; ++i) umma::mbar_init(&full[i], 1);
    umma::mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int jj) {  // chunk jj of this CTA's sequence -> stage jj % kPStage (one TMA box)
    int k, i;
    if (jj < nk0 * g.R0) {
      k = jj / g.R0;
      i = jj - k * g.R0;
    } else {
      const int j2 = jj - nk0 * g.R0;
      k = nk0 + j2 / R1;
      i = j2 - (k - nk0) * R1;
    }
    const int u = blockIdx.x + k * nblk;
    const bool fwd = u < P;
    const int pair = fwd ? u : u - P, r = fwd ? i : g.R - 1 - i;
    const int s = jj % kPStage;
    umma::mbar_expect_tx(&full[s], (uint32_t)kPRound * 2u);
    umma::tma_load_3d(ring + (size_t)s * (kPRound * 2), &tmK, 0, (g.first + r * kPRound) >> 6, pair, &full[s]);
  };
  if (tid == 0)
    for (int jj = 0; jj < min(kPStage, nchunks); ++jj) issue(jj);
  pdl_wait();  // tblg / pinfo come from the threshold kernel (sel: read by the previous step's attention,
  pdl_trigger();  // complete before the prep kernel triggered)
  A2ATS_TL(g_selc_tl, 2);
  // table of unit k: its compact words and (v*, m, K_eff, E) are staged into shared memory by
  // cp.async one unit ahead (no registers held, no stall at use); thread t < 4 W then
  // replicates word t >> 2 (two 16-B stores)
  __shared__ __align__(16) uint32_t sStage[2][256 + 4];
  const int tw = tid >> 2, tq = (tid & 3) * 2;
  auto pair_of = [&](int k) {
    const int u = blockIdx.x + k * nblk;
    return u < P ? u : u - P;
  };
  auto load_unit = [&](int k) {
    if (k >= nunit) return;
    const int pair = pair_of(k);
    uint32_t* st = sStage[k & 1];
    if (tid < W) {
      const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(st + tid));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(a.tblg + (size_t)pair * W + tid) : "memory");
    }
    if (tid == kPAll - 1) cp_async16(st + 256, a.pinfo + pair * 4);
    cp_async_commit();
  };
  auto unit_info = [&](int k) {  // after the staging of unit k is visible
    const uint32_t* st = sStage[k & 1];
    return PipeUnit{st[257], st[259] - st[257], st[258], 0u};  // m, D = E - m, cap = K_eff
  };
  auto store_table = [&](int k) {
    if (tw < W) {
      const uint32_t x = sStage[k & 1][tw];
      uint4* dst = reinterpret_cast<uint4*>(tbl0 + tw * 32);
      const uint4 v = make_uint4(x, x, x, x);
      dst[(tq + tw) & 7] = v;
      dst[(tq + 1 + tw) & 7] = v;
    }
  };
  load_unit(0);
  cp_async_wait<0>();
  __syncthreads();
  store_table(0);
  PipeUnit pu_cur = unit_info(0);
  __syncthreads();
  if (tid == 0) A2ATS_TLX(g_selc_tl, 4);
  int j = 0;
  ScanCtx c{a, g, (uint32_t)__cvta_generic_to_shared(ring), (uint32_t)__cvta_generic_to_shared(tbl0), full,
            &sTot[0][0], nchunks};
  for (int k = 0; k < nunit; ++k) {
    const int u = blockIdx.x + k * nblk;
    const bool fwd = u < P;
    load_unit(k + 1);
    auto expand = [&]() {
      if (k + 1 < nunit) {
        cp_async_wait<0>();
        __syncthreads();  // every thread's staged words
        store_table(k + 1);
      }
    };
    if (fwd) scan_unit<true>(c, 0, pair_of(k), g.R0, pu_cur, j, issue, expand);
    else scan_unit<false>(c, 0, pair_of(k), R1, pu_cur, j, issue, expand);
    __syncthreads();  // the next unit's table is visible
    if (k + 1 < nunit) pu_cur = unit_info(k + 1);
    if (tid == 0 && k == 0) A2ATS_TLX(g_selc_tl, 3);
  }
  A2ATS_TL(g_selc_tl, 1);
}

// ---------------------------------------------------------------- posting-list selection (f3)
// Inverted index: the tokens [0, n_post) of every pair grouped by code
// (post_off / post_tok, query-independent, built at prefill by a2ats_postings_build).  Since a
// token's approximate score is its code's (Eq. 21), the top-K set is the union of the lists of
// the codes above v* plus the first m tokens (by index) of the tied codes' lists (Q12): the
// step reads only those lists (about K entries per pair) instead of every code.  One CTA per
// pair: counts (hist - sinks/window) and the window-row logits before the dependency wait;
// v*, m from the registers (level_regs); the hit codes compacted into a table (list start,
// length, tied flag); a warp per hit code sets its list's candidate bits in the above or the
// tied bitmap; tokens [n_post, c1) not yet in the index are classified from their codes; then
// the bitmaps are scanned in token order (lanes on consecutive words, warp prefix of the
// counts): ascending emission with the tie quota, as in the code scan.
#ifndef A2ATS_QT_MINB
#define A2ATS_QT_MINB 4  // postings select CTAs per SM (tuning define)
#endif
constexpr int kQT = 256;             // postings select threads (16 codewords / thread, L <= 4096)
constexpr int kQWords = 16;          // bitmap words per thread per segment (4096-word segments)
constexpr int kQSurv = 512;          // survivors ranked directly (more: byte passes) -- keeps 4 CTAs / SM
constexpr int kQSinkMax = 64;        // list path: indexed sink tokens at most
constexpr int kQTiedMax = 8;         // list path: codes at v* at most (their lists are merged by rank)

// Block-wide exclusive scan of NV ints per thread (kQT threads): returns the exclusive prefix of
// each value and the block totals (in tot).  Ends synced; part[NV][kQT / 32] is scratch.
template <int NV>
__device__ __forceinline__ void q_scan(const int (&v)[NV], int (&ex)[NV], int (&tot)[NV], int (*part)[kQT / 32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) inc[i] = v[i];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int y = __shfl_up_sync(0xffffffffu, inc[i], off);
      if (lane >= off) inc[i] += y;
    }
  __syncthreads();  // part reusable
  if (lane == 31)
#pragma unroll
    for (int i = 0; i < NV; ++i) part[i][warp] = inc[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    ex[i] = inc[i] - v[i];
    tot[i] = 0;
    for (int w = 0; w < kQT / 32; ++w) {
      const int p = part[i][w];
      if (w < warp) ex[i] += p;
      tot[i] += p;
    }
  }
}

template <typename CT>  // code type: uint16_t, or uint8_t (code_bytes 1)
__global__ __launch_bounds__(kQT, A2ATS_QT_MINB) void select_postings_kernel(SelArgs a) {
  A2ATS_TL(g_sel_tl, 0);
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ SelShared S;
  __shared__ uint32_t s_cls[256];    // compact 2-bit classes (code >> 4), L <= 4096
  __shared__ int s_part[6][kQT / 32];  // (block scans of up to 6 values)
  __shared__ uint16_t s_sk[kQSinkMax];          // codes of the indexed sink tokens (list path)
  __shared__ int s_ts[kQTiedMax], s_tn[kQTiedMax];  // tied codes' lists (list path)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, pair = blockIdx.x;
  const int L4 = (a.L + 3) & ~3;
  // shared memory (small, so that four CTAs per SM leave most of the unified L1 to the loads):
  //   cnt [L4] | survivors skey, scnt [kQSurv each] | list bounds [LP]
  int* cnt = reinterpret_cast<int*>(sm);
  uint32_t* skey = sm + L4;
  int* scnt = reinterpret_cast<int*>(skey + kQSurv);
  int* orow = scnt + kQSurv;                                // the pair's list bounds (16-B aligned)
  const int R = L4 + 2 * kQSurv;                            // words dead after the level (cnt + survivors)
  const int ncand = max(0, a.c1 - a.c0), nwords = (ncand + 31) >> 5;
  const CT* cp = reinterpret_cast<const CT*>(sizeof(CT) == 1 ? static_cast<const void*>(a.codes8)
                                                              : static_cast<const void*>(a.codes)) +
                 (size_t)pair * a.n_max;
  const int32_t* ptok = a.post_tok + (size_t)pair * a.n_max;
  int32_t* selp = a.sel + (size_t)pair * a.sel_stride;
  const uint32_t cap = (uint32_t)a.keff;
  // list path: the index holds no window token and few sinks (the sinks of a list are its first
  // entries: lists are ascending)
  const int nsk = min(a.c0, a.n_post);
  const bool list_ok = a.n_post <= a.c1 && nsk <= kQSinkMax;
  float wacc[512 / kQT];
  if (a.wlog) {  // the pair's window-row logits (step inputs; scratch aliases the regions above)
    window_logits<kQT>(a, pair, reinterpret_cast<uint8_t*>(sm), wacc);
    __syncthreads();
  }
  // step inputs, every load in flight at once: the pair's hist row and list-bounds row (one bulk
  // copy each into shared memory when 16-B aligned, else coalesced loads), the codes of its sinks
  // / window tokens (not candidates: subtracted from hist), the indexed sinks' codes and the first
  // 4 kQT unindexed tail tokens' codes (registers)
  const int LP = postings_off_stride(a.L);
  const int post0 = pair * LP;
  uint32_t tcode[2], skmask = 0u;  // codes of tail tokens tb0 + 4 tid .. + 3 (16 bits each)
  {
    __shared__ __align__(8) uint64_t s_pbar;
    const int32_t* histp = a.hist + (size_t)pair * a.L;
    const bool bulk = (a.L & 3) == 0 && (reinterpret_cast<uintptr_t>(a.hist) & 15) == 0;
    if (bulk) {
      if (tid == 0) {
        umma::fence_proxy_async();  // (the window-logit scratch was written through the generic proxy)
        umma::mbar_init(&s_pbar, 1);
        umma::mbar_fence_init();
        umma::mbar_expect_tx(&s_pbar, (uint32_t)(a.L + LP) * 4u);
        umma::bulk_load(cnt, histp, (uint32_t)a.L * 4u, &s_pbar);
        umma::bulk_load(orow, a.post_off + post0, (uint32_t)LP * 4u, &s_pbar);
      }
    } else {
      for (int l = tid; l < a.L; l += kQT) cnt[l] = __ldg(histp + l);
      for (int i = tid; i <= a.L; i += kQT) orow[i] = __ldg(a.post_off + post0 + i);
    }
    const int nrem = a.n_s + max(0, a.hist_end - a.w0);  // (hist covers [0, hist_end))
    int rc = -1;
    if (tid < nrem) rc = cp[tid < a.n_s ? tid : a.w0 + (tid - a.n_s)];
    if (list_ok && tid < nsk) s_sk[tid] = cp[tid];
    if (tid == 0) {  // level_regs<.., PRE>: range and bins initialised here (before a barrier)
      S.s_kmin = 0xffffffffu;
      S.s_kmax = 0u;
    }
    S.bins[tid] = 0;  // (kQT == 256 bins)
    const int tb = max(a.n_post, a.c0) + 4 * tid;  // tail tokens tb .. tb + 3 (4 consecutive per thread)
#pragma unroll
    for (int r = 0; r < 2; ++r)
      tcode[r] = (tb + 2 * r < a.c1 ? (uint32_t)cp[tb + 2 * r] : 0u) |
                 (tb + 2 * r + 1 < a.c1 ? (uint32_t)cp[tb + 2 * r + 1] << 16 : 0u);
    A2ATS_TL(g_selp_tl, 0);
    __syncthreads();  // (barrier init, s_sk)
    for (int i = 0; i < nsk; ++i) {  // this thread's codewords holding an indexed sink
      const int code = s_sk[i];
      if ((code >> 4) == tid) skmask |= 1u << (code & 15);
    }
    if (bulk) umma::mbar_wait(&s_pbar, 0);
    if (rc >= 0) atomicSub(&cnt[rc], 1);
    for (int i = tid + kQT; i < nrem; i += kQT) atomicSub(&cnt[cp[i < a.n_s ? i : a.w0 + (i - a.n_s)]], 1);
    __syncthreads();
  }
  int c[16];
  load_c_regs<16>(a, cnt, c);
  A2ATS_TL(g_selp_tl, 1);
  pdl_wait();  // agg comes from the prep kernel
  pdl_trigger();
  A2ATS_TL(g_sel_tl, 2);
  if (a.wlog) store_window_logits<kQT>(a, pair, wacc);
  append_hist(a, pair, cp);
  if (a.keff <= 0) return;  // (uint8 codes: launched for the append's histogram alone)
  uint32_t k[16], kstar, m;
  level_regs<kQT, 16, true>(a, S, pair, c, k, skey, scnt, kQSurv, kstar, m);  // (ends synced: cnt dead)
  A2ATS_TL(g_sel_tl, 3);
  // classes of this thread's 16 codewords; hit codes (above or at v*, candidates present)
  int e_unused = 0;
  const uint32_t x = class_bits<16>(k, c, kstar, e_unused);
  s_cls[tid] = x;
  uint32_t hmask = 0u, tmask = 0u;
#pragma unroll
  for (int e = 0; e < 16; ++e)
    if (c[e] > 0 && k[e] <= kstar) {
      hmask |= 1u << e;
      if (k[e] == kstar) tmask |= 1u << e;
    }
  // bound e of this thread's 16 consecutive codewords (e <= 16; staged before the wait)
  auto bnd = [&](int e) { return orow[tid * 16 + e]; };
  A2ATS_TL(g_selp_tl, 2);
  const bool list_go = list_ok;
  // list path: sink entries at the head of a hit list (lists are ascending) are skipped
  auto skip_of = [&](int e) {
    if (!((skmask >> e) & 1u)) return 0;
    const int code = tid * 16 + e;
    int sk = 0;
    for (int i = 0; i < nsk; ++i) sk += s_sk[i] == code;
    return sk;
  };
  A2ATS_TL(g_selp_tl, 3);
  // block scans: [0] above codes, [1] above entries, [2] tied codes, [3] tied entries (list
  // path: entries past the sinks).  Hit codes visited bit by bit (no unrolled per-code copies:
  // the kernel stays small in the instruction cache)
  // short unindexed tails (<= 4 kQT tokens, 4 consecutive per thread from registers) are classified
  // here and ride on the same block scan: [4] tail above v*, [5] tail tied
  const int tb0 = max(a.n_post, a.c0);
  const bool short_tail = a.c1 - tb0 <= 4 * kQT;
  uint32_t tcl = 0u;  // 2-bit classes of this thread's 4 tail tokens
  int v[6] = {0, 0, 0, 0, 0, 0}, ex[6], tot[6];
  if (list_go && short_tail) {
    __syncthreads();  // (s_cls complete)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = tb0 + 4 * tid + j;
      if (t < a.c1) {
        const int l = (int)((tcode[j >> 1] >> (16 * (j & 1))) & 0xffffu);
        const uint32_t cl = (s_cls[l >> 4] >> (2 * (l & 15))) & 3u;
        tcl |= cl << (2 * j);
        v[4] += cl == 1u;
        v[5] += cl == 2u;
      }
    }
  }
  {
    int nAc = 0, nAe = 0, nTc = 0, nTe = 0;
    for (uint32_t mm = hmask; mm; mm &= mm - 1u) {
      const int e = __ffs(mm) - 1;
      const int n = bnd(e + 1) - bnd(e) - (list_go ? skip_of(e) : 0);
      if ((tmask >> e) & 1u) {
        ++nTc;
        nTe += n;
      } else {
        ++nAc;
        nAe += n;
      }
    }
    v[0] = nAc;
    v[1] = nAe;
    v[2] = nTc;
    v[3] = nTe;
  }
  q_scan<6>(v, ex, tot, s_part);
  A2ATS_TL(g_selp_tl, 4);
  const int nA = tot[0], A_idx = tot[1], nT = tot[2], E_idx = tot[3];
  const int RT = R + postings_off_stride(a.L);  // + the bounds row (dead once the tables are built)
  const int nA4 = (nA + 3) & ~3;
  if (list_go && 3 * nA4 <= R && nT <= kQTiedMax) {
    // ---- list path: the selection in index order (no ordered emission):
    //   [0, A_idx)        the above-v* codes' lists (code order; each ascending)
    //   [A_idx, A)        the above-v* tail tokens [n_post, c1) (ascending)
    //   [A, A + m)        the first m tied tokens in token order (tied lists merged, then the tail)
    int* hs = reinterpret_cast<int*>(sm);  // above code h: list start (past its sinks)
    int* hn = hs + nA4;                    //               entries
    int* hp = hn + nA4;                    //               output position
    // staging of the above entries at their output positions, 16-B phase of selp (bulk store)
    const int sph = (int)((reinterpret_cast<uintptr_t>(selp) >> 2) & 3);
    int* stg = hp + nA4 + sph;
    const int stg_cap = RT - 3 * nA4 - 4;
    {
      int ih = ex[0], ip = ex[1], it = ex[2];
      for (uint32_t mm = hmask; mm; mm &= mm - 1u) {
        const int e = __ffs(mm) - 1;
        const int st = bnd(e) + skip_of(e), n = bnd(e + 1) - st;
        if ((tmask >> e) & 1u) {
          s_ts[it] = st;
          s_tn[it] = n;
          ++it;
        } else {
          hs[ih] = st;
          hn[ih] = n;
          hp[ih] = ip;
          ++ih;
          ip += n;
        }
      }
    }
    __syncthreads();
    A2ATS_TL(g_selp_tl, 5);
    // above lists -> output.  Staged: every entry fetched by cp.async into shared memory at its
    // output position (one round trip for the whole selection), then coalesced stores.
    // Otherwise a warp per code (entries lane, lane + 32 loaded together), kU codes in flight.
    // one tied code: its first min(n, m) entries staged too (after the above entries), stored
    // once the tail's above count is known
    const int n_tie1 = nT == 1 ? min(s_tn[0], (int)m) : 0;
    // short tail: A (above count incl. the tail) is known, so the whole selection -- above lists,
    // tail tokens, the m ties -- is staged at its final positions and leaves by one bulk store
    const int A_s = A_idx + tot[4];
    const bool all_staged = short_tail && A_s + (int)m <= stg_cap;
    if (all_staged) {
      const int sub = lane & 7;
      for (int h = (warp << 2) + (lane >> 3); h < nA; h += (kQT / 32) * 4) {
        const int n = hn[h];
        const int32_t* src = ptok + hs[h] + sub;
        uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(stg + hp[h] + sub));
        int j = sub;
        for (; j + 24 < n; j += 32, src += 32, d += 128)
          asm volatile(
              "cp.async.ca.shared.global [%0], [%1], 4;\n\t"
              "cp.async.ca.shared.global [%2], [%3], 4;\n\t"
              "cp.async.ca.shared.global [%4], [%5], 4;\n\t"
              "cp.async.ca.shared.global [%6], [%7], 4;" ::"r"(d), "l"(src), "r"(d + 32), "l"(src + 8), "r"(d + 64),
              "l"(src + 16), "r"(d + 96), "l"(src + 24)
              : "memory");
        for (; j < n; j += 8, src += 8, d += 32)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
      }
      if (nT == 1)  // the tied list's first min(n, m) entries: tie indices 0 ..
        for (int j = tid; j < n_tie1; j += kQT) {
          const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(stg + A_s + j));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(ptok + s_ts[0] + j) : "memory");
        }
      // this thread's tail tokens: above ones after the lists, tied ones after the indexed ties
      {
        int pa = A_idx + ex[4], rt = E_idx + ex[5];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t cl = (tcl >> (2 * j)) & 3u;
          const int t = tb0 + 4 * tid + j;
          if (cl == 1u) stg[pa++] = t;
          if (cl == 2u) {
            if (rt < (int)m) stg[A_s + rt] = t;
            ++rt;
          }
        }
      }
      if (nT > 1)  // several tied codes: tie index of an entry = its rank in the merge of the lists
        for (int g = 0; g < nT; ++g) {
          const int st = s_ts[g], n = s_tn[g];
          for (int j = tid; j < n; j += kQT) {
            const int t = __ldg(ptok + st + j);
            int r = j;
            for (int g2 = 0; g2 < nT; ++g2) {
              if (g2 == g) continue;
              int lo = 0, hi = s_tn[g2];
              const int32_t* q2 = ptok + s_ts[g2];
              while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(q2 + mid) < t) lo = mid + 1;
                else hi = mid;
              }
              r += lo;
            }
            if (r < (int)m) stg[A_s + r] = t;
          }
        }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      const int lim = min(A_s + (int)m, (int)cap);
      const int i0 = min(lim, (4 - sph) & 3), i1 = i0 + ((lim - i0) & ~3);
      if (tid < i0) selp[tid] = stg[tid];
      if (tid < lim - i1) selp[i1 + tid] = stg[i1 + tid];
      if (tid == 0 && i1 > i0) {
        umma::fence_proxy_async();
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(selp + i0),
                     "r"(static_cast<uint32_t>(__cvta_generic_to_shared(stg + i0))), "r"((uint32_t)(i1 - i0) * 4u)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
      A2ATS_TL(g_selp_tl, 6);
      A2ATS_TL(g_selp_tl, 7);
      A2ATS_TL(g_sel_tl, 1);
      return;
    }
    const bool tie_staged = nT == 1 && A_idx + n_tie1 <= stg_cap;
    if (A_idx <= stg_cap) {
      const int sub = lane & 7;  // groups of 8 lanes, a code each (lists average N / L entries)
      for (int h = (warp << 2) + (lane >> 3); h < nA; h += (kQT / 32) * 4) {
        const int n = hn[h];
        const int32_t* src = ptok + hs[h] + sub;
        uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(stg + hp[h] + sub));
        int j = sub;
        for (; j + 24 < n; j += 32, src += 32, d += 128)
          asm volatile(
              "cp.async.ca.shared.global [%0], [%1], 4;\n\t"
              "cp.async.ca.shared.global [%2], [%3], 4;\n\t"
              "cp.async.ca.shared.global [%4], [%5], 4;\n\t"
              "cp.async.ca.shared.global [%6], [%7], 4;" ::"r"(d), "l"(src), "r"(d + 32), "l"(src + 8), "r"(d + 64),
              "l"(src + 16), "r"(d + 96), "l"(src + 24)
              : "memory");
        for (; j < n; j += 8, src += 8, d += 32)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
      }
      if (tie_staged)
        for (int j = tid; j < n_tie1; j += kQT) {
          const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(stg + A_idx + j));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(ptok + s_ts[0] + j) : "memory");
        }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      // out: the 16-B aligned middle by one bulk store (TMA engine), head / tail by threads
      const int lim = min(A_idx, (int)cap);
      const int i0 = min(lim, (4 - sph) & 3), i1 = i0 + ((lim - i0) & ~3);
      if (tid < i0) selp[tid] = stg[tid];
      if (tid < lim - i1) selp[i1 + tid] = stg[i1 + tid];
      if (tid == 0 && i1 > i0) {
        umma::fence_proxy_async();
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(selp + i0),
                     "r"(static_cast<uint32_t>(__cvta_generic_to_shared(stg + i0))), "r"((uint32_t)(i1 - i0) * 4u)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      constexpr int kU = 8, kW = kQT / 32;
      for (int h0 = warp; h0 < nA; h0 += kW * kU) {
        int tk[kU][2];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int h = h0 + u * kW;
          tk[u][0] = tk[u][1] = 0;
          if (h < nA) {
            const int st = hs[h], n = hn[h];
            if (lane < n) tk[u][0] = __ldg(ptok + st + lane);
            if (lane + 32 < n) tk[u][1] = __ldg(ptok + st + lane + 32);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int h = h0 + u * kW;
          if (h < nA) {
            const int st = hs[h], n = hn[h], p = hp[h];
            if (lane < n && (uint32_t)(p + lane) < cap) selp[p + lane] = tk[u][0];
            if (lane + 32 < n && (uint32_t)(p + lane + 32) < cap) selp[p + lane + 32] = tk[u][1];
            for (int j = 64 + lane; j < n; j += 32)
              if ((uint32_t)(p + j) < cap) selp[p + j] = __ldg(ptok + st + j);
          }
        }
      }
    }
    A2ATS_TL(g_selp_tl, 6);
    // tail [max(n_post, c0), c1): classified from codes; counts first (A needs the above count)
    auto tail_code = [&](int t, int) { return (int)cp[t]; };
    int tA = 0, tT = 0;
    for (int t = tb0 + tid, r = 0; t < a.c1; t += kQT, ++r) {
      const int l = tail_code(t, r);
      const uint32_t cl = (s_cls[l >> 4] >> (2 * (l & 15))) & 3u;
      tA += cl == 1u;
      tT += cl == 2u;
    }
    tA = __reduce_add_sync(0xffffffffu, tA);
    tT = __reduce_add_sync(0xffffffffu, tT);
    __syncthreads();
    if (lane == 0) {
      s_part[0][warp] = tA;
      s_part[1][warp] = tT;
    }
    __syncthreads();
    int A = A_idx;
    for (int w = 0; w < kQT / 32; ++w) A += s_part[0][w];
    if (tb0 < a.c1) {  // ordered compaction of the tail, kQT tokens per round
      int runA = A_idx, runT = 0;
      for (int base = tb0, r = 0; base < a.c1; base += kQT, ++r) {
        const int t = base + tid;
        uint32_t cl = 0u;
        if (t < a.c1) {
          const int l = tail_code(t, r);
          cl = (s_cls[l >> 4] >> (2 * (l & 15))) & 3u;
        }
        const int vv[2] = {cl == 1u, cl == 2u};
        int e2[2], t2[2];
        q_scan<2>(vv, e2, t2, s_part);
        if (cl == 1u && (uint32_t)(runA + e2[0]) < cap) selp[runA + e2[0]] = t;
        if (cl == 2u) {
          const int r = E_idx + runT + e2[1];  // tie index
          if (r < (int)m && (uint32_t)(A + r) < cap) selp[A + r] = t;
        }
        runA += t2[0];
        runT += t2[1];
      }
    }
    // the indexed ties: tie index of an entry = its rank in the merge of the tied lists
    if (tie_staged) {
      for (int j = tid; j < n_tie1; j += kQT)
        if ((uint32_t)(A + j) < cap) selp[A + j] = stg[A_idx + j];
    } else if (nT == 1) {
      const int st = s_ts[0];
      for (int j = tid; j < n_tie1; j += kQT)
        if ((uint32_t)(A + j) < cap) selp[A + j] = __ldg(ptok + st + j);
    } else {
      for (int g = 0; g < nT; ++g) {
        const int st = s_ts[g], n = s_tn[g];
        for (int j = tid; j < n; j += kQT) {
          const int t = __ldg(ptok + st + j);
          int r = j;
          for (int g2 = 0; g2 < nT; ++g2) {
            if (g2 == g) continue;
            int lo = 0, hi = s_tn[g2];  // #entries of list g2 below t
            const int32_t* q2 = ptok + s_ts[g2];
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (__ldg(q2 + mid) < t) lo = mid + 1;
              else hi = mid;
            }
            r += lo;
          }
          if (r < (int)m && (uint32_t)(A + r) < cap) selp[A + r] = t;
        }
      }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // (the bulk store complete)
    A2ATS_TL(g_selp_tl, 7);
    A2ATS_TL(g_sel_tl, 1);
    return;
  }
  // ---- bitmap path (sinks / window tokens in the index, or very many hit / tied codes):
  // candidate bits in an above and a tied bitmap, then an ordered emission over the bitmaps
  const int nhit = nA + nT, hcap = R / 2;
  int* hs = reinterpret_cast<int*>(sm);  // hit code h: list start
  int* hl = hs + hcap;                   //             length | bit 31 if tied at v*
  // above-v* and tied bitmaps of the candidates: the pair's workspace slice (global memory)
  const int nw4 = (nwords + 3) & ~3;
  uint32_t* bab = a.pbits + (size_t)pair * a.pbits_stride;
  uint32_t* bti = bab + nw4;
  for (int i = tid; i < 2 * nw4; i += kQT) bab[i] = 0u;
  int bh = ex[0] + ex[2];
  const bool in_smem = nhit <= hcap;
  if (in_smem) {
    for (uint32_t mm = hmask; mm; mm &= mm - 1u) {
      const int e = __ffs(mm) - 1;
      hs[bh] = bnd(e);
      hl[bh] = (bnd(e + 1) - bnd(e)) | ((((x >> (2 * e)) & 3u) == 2u) ? (int)0x80000000 : 0);
      ++bh;
    }
  }
  __syncthreads();
  A2ATS_TL(g_selp_tl, 5);
  // list entries -> candidate bits (entries outside [c0, c1) are sinks / window): a warp per hit
  // code, lanes over its list (entries lane, lane + 32 loaded together); kU codes per warp in
  // flight; longer lists loop
  auto set_bit = [&](int t, bool tied) {
    if (t >= a.c0 && t < a.c1) atomicOr((tied ? bti : bab) + ((t - a.c0) >> 5), 1u << ((t - a.c0) & 31));
  };
  if (in_smem) {
    constexpr int kU = 8, kW = kQT / 32;
    for (int h0 = warp; h0 < nhit; h0 += kW * kU) {
      int tk[kU][2];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int h = h0 + u * kW;
        tk[u][0] = tk[u][1] = -1;
        if (h < nhit) {
          const int st = hs[h], len = hl[h] & 0x7fffffff;
          if (lane < len) tk[u][0] = __ldg(ptok + st + lane);
          if (lane + 32 < len) tk[u][1] = __ldg(ptok + st + lane + 32);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int h = h0 + u * kW;
        if (h < nhit) {
          const int st = hs[h], len = hl[h] & 0x7fffffff;
          const bool tied = hl[h] < 0;
          set_bit(tk[u][0], tied);
          set_bit(tk[u][1], tied);
          for (int j = 64 + lane; j < len; j += 32) set_bit(__ldg(ptok + st + j), tied);
        }
      }
    }
  } else {  // very many hit codes (ties across much of the codebook): thread per hit codeword
#pragma unroll 1
    for (int e = 0; e < 16; ++e) {
      if (!((hmask >> e) & 1u)) continue;
      const bool tied = ((x >> (2 * e)) & 3u) == 2u;
      const int l = tid * 16 + e, i1 = __ldg(a.post_off + post0 + l + 1);
      for (int i = __ldg(a.post_off + post0 + l); i < i1; ++i) set_bit(__ldg(ptok + i), tied);
    }
  }
  A2ATS_TL(g_selp_tl, 6);
  // tokens not yet in the index: classified from their codes
  for (int t = max(a.n_post, a.c0) + tid; t < a.c1; t += kQT) {
    const int l = cp[t];
    const uint32_t cl = (s_cls[l >> 4] >> (2 * (l & 15))) & 3u;
    if (cl) set_bit(t, cl == 2u);
  }
  __syncthreads();
  A2ATS_TL(g_selp_tl, 7);
  // ordered emission.  Segments of kQT * kQWords words; warp w takes words [512 w, 512 w + 512)
  // of the segment, lane l word 32 i + l at step i (consecutive lanes: consecutive words and
  // nearby output positions).  Selected bits of a word: the above-v* bits and the tied bits of
  // tie index < m; they go, in token order, to #above-before + min(#tied-before, m) onwards.
  uint32_t run_gt = 0u, run_eq = 0u;
  for (int seg = 0; seg < nwords; seg += kQT * kQWords) {
    const int wb = seg + warp * (32 * kQWords);
    uint32_t ng = 0u, ne = 0u;
#pragma unroll
    for (int i = 0; i < kQWords; ++i) {
      const int w = wb + 32 * i + lane;
      if (w < nwords) {
        ng += __popc(bab[w]);
        ne += __popc(bti[w]);
      }
    }
    ng = __reduce_add_sync(0xffffffffu, ng);
    ne = __reduce_add_sync(0xffffffffu, ne);
    __syncthreads();  // the previous segment's s_part reads are done
    if (lane == 0) {
      s_part[0][warp] = ng;
      s_part[1][warp] = ne;
    }
    __syncthreads();
    uint32_t gb = run_gt, eb = run_eq, tg = 0u, te = 0u;
    for (int w = 0; w < kQT / 32; ++w) {
      const uint32_t pg = s_part[0][w], pe = s_part[1][w];
      if (w < warp) {
        gb += pg;
        eb += pe;
      }
      tg += pg;
      te += pe;
    }
#pragma unroll 1
    for (int i = 0; i < kQWords; ++i) {
      const int w = wb + 32 * i + lane;
      if (wb + 32 * i >= nwords) break;  // (warp-uniform)
      uint32_t A = 0u, T = 0u;
      if (w < nwords) {
        A = bab[w];
        T = bti[w];
      }
      const uint32_t pa = __popc(A), pt = __popc(T);
      uint32_t incl = pa | (pt << 16);  // <= 32 * 32 per field
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t ab = gb + (incl & 0xffffu) - pa, tb_ = eb + (incl >> 16) - pt;
      if (T) {  // keep the tied bits of tie index < m (all, none, or a prefix at the boundary)
        const uint32_t keep = m > tb_ ? m - tb_ : 0u;
        for (uint32_t d = pt > keep ? pt - keep : 0u; d > 0u; --d) T &= ~(0x80000000u >> __clz(T));
      }
      uint32_t S = A | T, pos = ab + min(tb_, m);
      const int tok0 = a.c0 + w * 32;
      while (S) {
        const int bit = __ffs(S) - 1;
        S &= S - 1u;
        if (pos < cap) selp[pos] = tok0 + bit;
        ++pos;
      }
      gb += tot & 0xffffu;
      eb += tot >> 16;
    }
    run_gt += tg;
    run_eq += te;
  }
  A2ATS_TL(g_sel_tl, 1);
}


// Inverted index of tokens [0, n_tok) per pair, every list ascending (deterministic): warp w
// owns the contiguous tokens [w n / kBW, (w + 1) n / kBW); per-(warp, code) counts -> cursors
// (code-major exclusive prefix: post_off, then the warps in order) -> each warp places its
// tokens in order, 32 per step, ranks among equal codes of a step from match_any.
constexpr int kBW = 8;
template <typename CT>
__global__ __launch_bounds__(kBW * 32) void postings_build_kernel(const CT* __restrict__ codes, int n_max, int L,
                                                                  int n_tok, int32_t* __restrict__ post_off,
                                                                  int32_t* __restrict__ post_tok) {
  extern __shared__ __align__(16) int pcnt[];  // [kBW][L]: counts, then cursors
  __shared__ int s_w[kBW];
  constexpr int NT = kBW * 32;
  const int pair = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const CT* cp = codes + (size_t)pair * n_max;
  for (int i = tid; i < kBW * L; i += NT) pcnt[i] = 0;
  __syncthreads();
  const int per = (n_tok + kBW - 1) / kBW, t0 = min(n_tok, warp * per), t1 = min(n_tok, t0 + per);
  int* my = pcnt + warp * L;
  for (int tb = t0; tb < t1; tb += 32 * 8) {  // 8 code loads in flight per lane
    int cc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = tb + 32 * k + lane;
      cc[k] = t < t1 ? (int)cp[t] : -1;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (cc[k] >= 0) atomicAdd(&my[cc[k]], 1);
  }
  __syncthreads();
  // thread owns codes [l0, l0 + pc): its total, block scan, then the cursors
  const int pc = (L + NT - 1) / NT, l0 = tid * pc;
  int s = 0;
  for (int i = 0; i < pc && l0 + i < L; ++i)
    for (int w = 0; w < kBW; ++w) s += pcnt[w * L + l0 + i];
  int incl = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int base = incl - s, total = 0;
  for (int w = 0; w < kBW; ++w) {
    if (w < warp) base += s_w[w];
    total += s_w[w];
  }
  int32_t* offp = post_off + (size_t)pair * postings_off_stride(L);
  for (int i = 0; i < pc && l0 + i < L; ++i) {
    offp[l0 + i] = base;
    for (int w = 0; w < kBW; ++w) {
      const int cnt = pcnt[w * L + l0 + i];
      pcnt[w * L + l0 + i] = base;
      base += cnt;
    }
  }
  if (tid == 0) offp[L] = total;
  __syncthreads();
  int32_t* tp = post_tok + (size_t)pair * n_max;
  const unsigned lt = (1u << lane) - 1u;
  for (int tb0 = t0; tb0 < t1; tb0 += 32 * 8) {  // 8 code loads in flight per lane, then 8 steps of 32
    int cc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = tb0 + 32 * k + lane;
      cc[k] = t < t1 ? (int)cp[t] : -1 - lane;  // (inactive lanes: unique keys)
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = tb0 + 32 * k + lane, code = cc[k];
      const unsigned peers = __match_any_sync(0xffffffffu, code);
      int b = 0;
      if (t < t1) {
        b = my[code];
        tp[b + __popc(peers & lt)] = t;
      }
      __syncwarp();
      if (t < t1 && (peers & lt) == 0u) my[code] = b + __popc(peers);
      __syncwarp();
    }
  }
}

size_t shard_thresh_smem_bytes(int L) { return (size_t)((L + 3) & ~3) * 8 + 2 * kTSurv * 4; }
size_t thresh_smem_bytes(int L) { return (size_t)((L + 3) & ~3) * 4 + 2 * kTSurv * 4; }  // cnt + survivors
size_t scan_smem_bytes(int) { return 32768 + 32768 + (size_t)kPStage * kPRound * 2; }  // align slack + table + ring


template <int MODE>
__device__ __forceinline__ void select_body(const SelArgs& a) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ SelShared S;
  int* cnt = reinterpret_cast<int*>(sm);  // [L]
  uint32_t* key = sm + ((a.L + 3) & ~3);  // [L], 16-B aligned
  uint32_t* tbl = sm;                     // [W*32], aliases cnt/key once they are dead
  const int tbl_words = (max(((a.L + 3) & ~3) + a.L, a.W * 32) + 3) / 4 * 4;
  uint32_t* skey = sm + tbl_words;                                   // [kSurvCap] (find_level modes)
  int* scnt = reinterpret_cast<int*>(skey + kSurvCap);              // [kSurvCap]
  uint4* sC = reinterpret_cast<uint4*>(sm + tbl_words + (ModeTraits<MODE>::surv ? 2 * kSurvCap : 0));  // [kCH / 8]
  if (MODE == kThresh || MODE == kScanC) {
    split_body<MODE>(a, S, cnt, key, tbl, skey, scnt, sC);
    return;
  }

  const int tid = threadIdx.x;
  const int pair = blockIdx.x;
  const int lo = a.shard_begin, hi = a.shard_begin + a.shard_len;
  const uint16_t* cp_local = a.codes + (size_t)pair * a.n_max;  // local index = global - lo
  const int c0 = max(a.c0, lo), c1 = min(a.c1, hi);             // local part of the candidate range
  A2ATS_PHASE(g_sel_phase, 0);

  // kFused: step inputs first (overlapping the previous kernel's tail):
  // the first chunk of local candidate codes, and (fused) the candidate counts
  const int first = lo + (((c0 - lo) >> 3) << 3);
  if (c0 < c1) prefetch_chunk(a, cp_local, first, c1, sC);
  // L <= 8 * kNT: every thread keeps 8 codewords' counts and keys in registers (level_regs)
  const bool regs = (MODE == kFused) && a.L <= 8 * kNT;
  int c8[8];
  if (MODE == kFused) load_cnt(a, pair, cnt, cp_local);
  if (regs) load_c_regs<8>(a, cnt, c8);
  A2ATS_PHASE(g_sel_phase, 1);
  pdl_wait();  // agg comes from the LUT kernel
  pdl_trigger();
  uint32_t kstar, m, cap;
  int32_t* selp = a.sel + (size_t)pair * a.sel_stride;
  if (MODE == kFused) {
    if (a.keff == 0) {  // nothing to select (launched for the histogram update only)
      cp_async_wait<0>();
      append_hist(a, pair, cp_local);
      return;
    }
    if (regs) {
      uint32_t k8[8];
      level_regs<kNT, 8>(a, S, pair, c8, k8, skey, scnt, kSurvCap, kstar, m);
      // class table: word w = codewords of threads 2w (low half) and 2w + 1, replicated 32x
      int e_unused = 0;
      const uint32_t x = class_bits<8>(k8, c8, kstar, e_unused);
      const uint32_t o = __shfl_xor_sync(0xffffffffu, x, 1);
      const uint32_t xw = (tid & 1) ? (o | (x << 16)) : (x | (o << 16));
      const int w = tid >> 1;
      if (w < a.W) {
        uint4* dst = reinterpret_cast<uint4*>(tbl + w * 32);
        const uint4 v = make_uint4(xw, xw, xw, xw);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[((tid & 1) * 4 + q + w) & 7] = v;
      }
      __syncthreads();
    } else {
      load_keys(a, S, pair, cnt, key);
      A2ATS_PHASE(g_sel_phase, 2);
      find_level(a, S, cnt, key, a.keff, skey, scnt);
      A2ATS_PHASE(g_sel_phase, 5);
      kstar = S.s_kstar;
      m = S.s_m;
    }
    cap = (uint32_t)a.keff;
  }
  if (!regs) build_table(a, key, kstar, tbl);
  A2ATS_PHASE(g_sel_phase, 6);
  scan_emit(a, S, tbl, cp_local, c0, c1, m, cap, selp, sC);
  A2ATS_PHASE(g_sel_phase, 7);
  if (MODE == kFused) append_hist(a, pair, cp_local);
}

template <int MODE>
__global__ __launch_bounds__(kNT, ModeTraits<MODE>::min_blocks) void select_kernel(SelArgs a) {
  if (MODE == kScanC) {
    A2ATS_TL(g_selc_tl, 0);
  } else {
    A2ATS_TL(g_sel_tl, 0);
  }
  select_body<MODE>(a);
  if (MODE == kScanC) {
    A2ATS_TL(g_selc_tl, 1);
  } else {
    A2ATS_TL(g_sel_tl, 1);
  }
}

template <int MODE>
cudaError_t launch_mode(const SelArgs& a, int P, cudaStream_t st) {  // P: CTAs
  const int tbl_words = (max(((a.L + 3) & ~3) + a.L, a.W * 32) + 3) / 4 * 4;
  const int smem = tbl_words * 4 + (ModeTraits<MODE>::surv ? 2 * kSurvCap * 4 : 0) +
                   (ModeTraits<MODE>::codes ? kCH * 2 : 0) + ModeTraits<MODE>::extra;
  cudaError_t e = ensure_smem(select_kernel<MODE>, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(select_kernel<MODE>, dim3(P), dim3(kNT), smem, st, a);
}
}  // namespace

cudaError_t launch_select(const SelArgs& a, int P, cudaStream_t st) { return launch_mode<kFused>(a, P, st); }

cudaError_t launch_select_split(const SelArgs& a, int P, cudaStream_t st) {
  cudaError_t e = launch_mode<kThresh>(a, P, st);
  if (e != cudaSuccess) return e;
  return launch_mode<kScanC>(a, P * a.nchunk, st);
}
int select_chunk_tokens() { return kCH; }

bool select_pipe_ok(int L) { return L <= 4096; }

size_t postings_smem_bytes(int L, bool window) {
  const size_t base = (size_t)((L + 3) & ~3) * 4 + 2 * kQSurv * 4 + (size_t)postings_off_stride(L) * 4;
  return window ? std::max(base, (size_t)kWinScratch) : base;
}
bool select_postings_ok(int L, int) { return L <= 4096; }

template <typename CT>
cudaError_t launch_select_postings_t(const SelArgs& a, cudaStream_t st) {
  const int smem = (int)postings_smem_bytes(a.L, a.wlog != nullptr);
  cudaError_t e = ensure_smem(select_postings_kernel<CT>, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(select_postings_kernel<CT>, dim3(a.P), dim3(kQT), smem, st, a);
}
cudaError_t launch_select_postings(const SelArgs& a, cudaStream_t st) {
  return a.codes8 ? launch_select_postings_t<uint8_t>(a, st) : launch_select_postings_t<uint16_t>(a, st);
}

template <typename CT>
cudaError_t launch_postings_build_t(const CT* codes, int P, int n_max, int L, int n_tok, int32_t* post_off,
                                    int32_t* post_tok, cudaStream_t st) {
  const int smem = kBW * L * 4;
  cudaError_t e = ensure_smem(postings_build_kernel<CT>, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(postings_build_kernel<CT>, dim3(P), dim3(kBW * 32), smem, st, codes, n_max, L, n_tok, post_off,
                    post_tok);
}
cudaError_t launch_postings_build(const uint16_t* codes, bool codes8, int P, int n_max, int L, int n_tok,
                                  int32_t* post_off, int32_t* post_tok, cudaStream_t st) {
  return codes8 ? launch_postings_build_t(reinterpret_cast<const uint8_t*>(codes), P, n_max, L, n_tok, post_off,
                                          post_tok, st)
                : launch_postings_build_t(codes, P, n_max, L, n_tok, post_off, post_tok, st);
}

cudaError_t launch_select_shard(const SelArgs& a, const CUtensorMap& tmK, int nblk, cudaStream_t st) {
  if (!select_pipe_ok(a.L)) return cudaErrorInvalidValue;
  const int smt = (int)std::max(shard_thresh_smem_bytes(a.L), a.wlog ? (size_t)kWinScratch : (size_t)0);
  const int sms = (int)scan_smem_bytes(a.W);
  cudaError_t e = ensure_smem(select_shard_thresh_kernel, smt);
  if (e != cudaSuccess) return e;
  e = ensure_smem(select_scan_kernel, sms);
  if (e != cudaSuccess) return e;
  e = launch_pdl(select_shard_thresh_kernel, dim3(a.P), dim3(kTT), smt, st, a);
  if (e != cudaSuccess || nblk <= 0) return e;
  return launch_pdl(select_scan_kernel, dim3(nblk), dim3(kPAll), sms, st, tmK, a);
}

cudaError_t launch_select_pipe(const SelArgs& a, const CUtensorMap& tmK, int nblk, cudaStream_t st) {
  if (!select_pipe_ok(a.L)) return cudaErrorInvalidValue;
  const int smt = (int)std::max(thresh_smem_bytes(a.L), a.wlog ? (size_t)kWinScratch : (size_t)0);
  const int sms = (int)scan_smem_bytes(a.W);
  cudaError_t e = ensure_smem(select_thresh_kernel, smt);
  if (e != cudaSuccess) return e;
  e = ensure_smem(select_scan_kernel, sms);
  if (e != cudaSuccess) return e;
  e = launch_pdl(select_thresh_kernel, dim3(a.P), dim3(kTT), smt, st, a);
  if (e != cudaSuccess) return e;
  return launch_pdl(select_scan_kernel, dim3(nblk), dim3(kPAll), sms, st, tmK, a);
}


}  // namespace a2ats

A2ATS_PHASE_EXPORT(a2ats_debug_select_phases, a2ats::g_sel_phase)
A2ATS_TL_EXPORT(a2ats_debug_select_timeline, a2ats::g_sel_tl)
A2ATS_TL_EXPORT(a2ats_debug_selc_timeline, a2ats::g_selc_tl)
A2ATS_TL_EXPORT(a2ats_debug_selp_timeline, a2ats::g_selp_tl)
