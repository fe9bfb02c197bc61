// a3 + a4: approximate scores through the code stream and exact top-K selection.
//
// Scores take only L distinct values per (b, KV head) pair (u^_t = LUT[s_t],
// Eq. 21), so the K-th largest score is found by a count-weighted
// radix select over the L codewords, not over the N tokens.  One CTA owns one
// pair:
//
//  1. candidate histogram over codewords: the caller-maintained hist minus the
//     sink/window codes (the code stream is then read exactly once), or,
//     without hist, an extra pass over the codes;
//  2. count-weighted selection of the K-th largest agg level v*: a weighted
//     histogram over 256 equal-width key bins finds the bin holding the K-th
//     token, its (few) codewords are compacted and the exact key is resolved by
//     single-warp radix passes; tie quota m = K - #{agg > v*};
//  3. 2-bit class per codeword (1: agg > v*, 2: agg == v*), replicated 32x in
//     shared memory so lane l reads bank l (conflict-free gather by code);
//  4. stream the codes chunk by chunk (prefetched into registers), classify each
//     token, and write the selected indices in ascending order (block scan +
//     running prefix).  A token with agg == v* is kept iff fewer than m such
//     tokens precede it: the lowest-index tie-break of reading Q12.
//
// The same phases serve the sequence-sharded step: shard_hist
// (local candidate histogram), shard_thresh (v*, m from the all-reduced
// histogram + this rank's above/at counts) and shard_scan (local emission with
// the rank's tie quota, from the all-gathered counts).
#include "internal.cuh"

namespace a2ats {

namespace {
A2ATS_TL_DECL(g_sel_tl)
A2ATS_PHASE_DECL(g_sel_phase)

constexpr int kNT = 512;             // threads per CTA
constexpr int kNW = kNT / 32;
constexpr int kVPT = 8;              // 128-bit code loads per thread per chunk
constexpr int kCH = kNT * kVPT * 8;  // tokens per chunk (32768)
constexpr int kSurvCap = 2048;       // survivor list capacity of the single-warp radix passes

enum SelMode { kFused = 0, kShardHist = 1, kShardThresh = 2, kShardScan = 3 };

__device__ __forceinline__ uint32_t spread16(uint32_t v) {
  v &= 0xffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

struct SelShared {
  int bins[256];
  uint32_t cls[1024];    // compact 2-bit classes (W <= 1024)
  uint32_t wsum[kVPT][kNW];
  uint32_t wsum_total;
  uint32_t skey[kSurvCap];
  int scnt[kSurvCap];
  int s_digit, s_kk, s_nsurv;
  uint32_t s_and, s_or, s_kstar, s_m;
  uint32_t s_run[2];
};

// Load the per-codeword candidate counts and ordered keys of one pair into smem.
//   cnt[l] = hist[l] - #(local sink/window tokens with code l)   (hist given)
//          = #(local candidate tokens with code l)                (otherwise)
// key[l] = ~ordered(agg[l]) (ascending key = descending agg).
__device__ void load_counts(const SelArgs& a, int pair, int* cnt, uint32_t* key, const uint16_t* cp_local) {
  const int tid = threadIdx.x;
  const float* aggp = a.agg + (size_t)pair * a.L;
  const int32_t* histp = a.hist ? a.hist + (size_t)pair * a.L : nullptr;
  for (int base = 0; base < a.L; base += 8 * kNT) {  // all loads of a batch in flight before use
    float av[8];
    int hv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int l = base + i * kNT + tid;
      av[i] = l < a.L ? __ldg(aggp + l) : 0.f;
      hv[i] = (histp && l < a.L) ? __ldg(histp + l) : 0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int l = base + i * kNT + tid;
      if (l < a.L) {
        cnt[l] = hv[i];
        key[l] = ~ordered_key(av[i]);
      }
    }
  }
  __syncthreads();
  const int lo = a.shard_begin, hi = a.shard_begin + a.shard_len;  // local global-index range
  if (a.hist) {
    // remove the local sinks [0, n_s) and window [w0, n_ctx): they are not candidates
    const int nrem = a.n_s + (a.n_ctx - a.w0);
    for (int i = tid; i < nrem; i += kNT) {
      const int t = i < a.n_s ? i : a.w0 + (i - a.n_s);
      if (t >= lo && t < hi) atomicSub(&cnt[cp_local[t - lo]], 1);
    }
  } else {
    const int c0 = max(a.c0, lo), c1 = min(a.c1, hi);
    if (c0 < c1) {
      const int v0 = (c0 - lo) >> 3, v1 = (c1 - lo + 7) >> 3;
      for (int vi = v0 + tid; vi < v1; vi += kNT) {
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
  __syncthreads();
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

// Count-weighted selection of the keff-th smallest key over cnt/key (all threads).
// Result in S.s_kstar (key of v*) and S.s_m (tie quota, >= 1).
__device__ void radix_kth(const SelArgs& a, SelShared& S, const int* cnt, const uint32_t* key, int keff) {
  // 1. key range of the candidates; 2. weighted histogram over 256 equal-width key
  //    bins (monotone in the key, so in agg) to find the bin holding the K-th
  //    token; 3. compact that bin's codewords (typically tens) and resolve the
  //    exact K-th key with single-warp radix passes over them.  Few block barriers:
  //    this runs once per CTA on the critical path.
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    S.s_and = 0xffffffffu;  // min key
    S.s_or = 0u;            // max key
    S.s_nsurv = 0;
  }
  for (int i = tid; i < 256; i += kNT) S.bins[i] = 0;
  __syncthreads();
  uint32_t kmn = 0xffffffffu, kmx = 0u;
  for (int l = tid; l < a.L; l += kNT) {
    if (cnt[l] > 0) {
      kmn = min(kmn, key[l]);
      kmx = max(kmx, key[l]);
    }
  }
  kmn = __reduce_min_sync(0xffffffffu, kmn);
  kmx = __reduce_max_sync(0xffffffffu, kmx);
  if (lane == 0) {
    atomicMin(&S.s_and, kmn);
    atomicMax(&S.s_or, kmx);
  }
  __syncthreads();
  A2ATS_PHASE(g_sel_phase, 2);
  kmn = S.s_and;
  kmx = S.s_or;
  if (kmn == kmx) {  // a single level holds every candidate
    if (tid == 0) {
      S.s_kstar = kmn;
      S.s_m = (uint32_t)keff;
    }
    __syncthreads();
    return;
  }
  // 256 bins of equal width in agg VALUE over [amin, amax], ascending bin = descending
  // agg (monotone and deterministic: one subtract, one multiply, one truncation).
  // Equal-width bins in key space would be one binade wide and hold hundreds of codes.
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
  for (int l = tid; l < a.L; l += kNT) {
    const int c = cnt[l];
    if (c > 0) atomicAdd(&S.bins[bin_of(key[l])], c);
  }
  __syncthreads();
  if (warp == 0) pick_digit(S, keff);
  __syncthreads();
  A2ATS_PHASE(g_sel_phase, 3);
  const int bstar = S.s_digit;
  int kk = S.s_kk;
  {
    // survivors = candidate codewords of bin b*; one shared atomic per warp
    int nkeep = 0;
    for (int l0 = 0; l0 < a.L; l0 += kNT) {
      const int l = l0 + tid;
      nkeep += __popc(__ballot_sync(0xffffffffu, l < a.L && cnt[l] > 0 && bin_of(key[l]) == bstar));
    }
    int base = 0;
    if (lane == 0 && nkeep) base = atomicAdd(&S.s_nsurv, nkeep);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int l0 = 0; l0 < a.L; l0 += kNT) {
      const int l = l0 + tid;
      const bool keep = l < a.L && cnt[l] > 0 && bin_of(key[l]) == bstar;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int slot = base + __popc(bal & ((1u << lane) - 1u));
        if (slot < kSurvCap) {
          S.skey[slot] = key[l];
          S.scnt[slot] = cnt[l];
        }
      }
      base += __popc(bal);
    }
  }
  __syncthreads();
  A2ATS_PHASE(g_sel_phase, 4);
  const int nsurv = S.s_nsurv;
  if (nsurv <= kSurvCap) {
    if (warp == 0) {
      // exact K-th key among the survivors: radix passes from their first differing bit
      uint32_t sa = 0xffffffffu, so = 0u;
      for (int i = lane; i < nsurv; i += 32) {
        sa &= S.skey[i];
        so |= S.skey[i];
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
            const uint32_t k = S.skey[i];
            if ((k & mask) == prefix) atomicAdd(&S.bins[(k >> shift) & 255u], S.scnt[i]);
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
    __syncthreads();
    return;
  }
  // degenerate value distributions (more survivors than the list holds): block-wide
  // byte passes restricted to bin b*
  uint32_t prefix = 0, mask = 0;
  for (int pass = 3; pass >= 0; --pass) {
    const int shift = 8 * pass;
    for (int i = tid; i < 256; i += kNT) S.bins[i] = 0;
    __syncthreads();
    for (int l = tid; l < a.L; l += kNT) {
      const int c = cnt[l];
      const uint32_t k = key[l];
      if (c > 0 && bin_of(k) == bstar && (k & mask) == prefix) atomicAdd(&S.bins[(k >> shift) & 255u], c);
    }
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
  __syncthreads();
}

// 2-bit classes vs kstar, compact then replicated 32x into tbl (may alias key/cnt).
__device__ void build_table(const SelArgs& a, SelShared& S, const uint32_t* key, uint32_t kstar, uint32_t* tbl) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int gi = warp; gi < (a.L + 31) / 32; gi += kNW) {
    const int l = gi * 32 + lane;
    uint32_t c = 0;
    if (l < a.L) {
      const uint32_t k = key[l];
      c = (k < kstar) ? 1u : ((k == kstar) ? 2u : 0u);
    }
    const uint32_t gtm = __ballot_sync(0xffffffffu, c == 1u);
    const uint32_t eqm = __ballot_sync(0xffffffffu, c == 2u);
    if (lane < 2 && gi * 2 + lane < a.W) {
      const uint32_t g16 = lane ? (gtm >> 16) : gtm, e16 = lane ? (eqm >> 16) : eqm;
      S.cls[gi * 2 + lane] = spread16(g16) | (spread16(e16) << 1);
    }
  }
  __syncthreads();
  for (int i = tid; i < a.W * 32; i += kNT) tbl[i] = S.cls[i >> 5];
  __syncthreads();
}

// Stream the local candidate codes, emit the selected token indices (global) in
// ascending order: every token above v*, plus the first m tied tokens.
// v[] holds the prefetched first chunk.  Returns the number emitted.
__device__ uint32_t scan_emit(const SelArgs& a, SelShared& S, const uint32_t* tbl, const uint16_t* cp_local, int c0,
                              int c1, uint32_t m, uint32_t cap, int32_t* selp, const uint4* sC, uint32_t* sPk,
                              uint32_t* sIn) {
  // Compact loops throughout (no full unrolling): this code runs once per CTA, and
  // straight-line SASS of that size stalls on instruction fetch.
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lo = a.shard_begin;
  const int first = lo + (((c0 - lo) >> 3) << 3);  // 8-aligned (local index) start
  const int nchunk = c1 > c0 ? (c1 - first + kCH - 1) / kCH : 0;
  if (tid == 0) {
    S.s_run[0] = 0;
    S.s_run[1] = 0;
  }
  for (int ch = 0; ch < nchunk; ++ch) {
    const int cb = first + ch * kCH;
    cp_async_wait<0>();  // this chunk's codes (prefetched with cp.async) are in sC
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < kVPT; ++j) {
      const int t0 = cb + (j * kNT + tid) * 8;
      const uint4 x = sC[j * kNT + tid];
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
      uint32_t p = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t code = (w[e >> 1] >> ((e & 1) * 16)) & 0xffffu;
        const uint32_t word = tbl[((code >> 4) << 5) + lane];
        p |= ((word >> ((code & 15u) * 2u)) & 3u) << (2 * e);
      }
      if (t0 < c0 || t0 + 8 > c1) {
        uint32_t mk = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (t0 + e >= c0 && t0 + e < c1) mk |= 3u << (2 * e);
        p &= mk;
      }
      const uint32_t pk = (uint32_t)__popc(p & 0x5555u) | ((uint32_t)__popc(p & 0xaaaau) << 16);
      uint32_t x2 = pk;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x2, off);
        if (lane >= off) x2 += y;
      }
      if (lane == 31) S.wsum[j][warp] = x2;
      sPk[j * kNT + tid] = p;
      sIn[j * kNT + tid] = x2 - pk;  // exclusive within the warp
    }
    __syncthreads();
    if (ch + 1 < nchunk) {  // sC is free: prefetch the next chunk during scan + emission
      for (int j = 0; j < kVPT; ++j) {
        const int t0 = cb + kCH + (j * kNT + tid) * 8;
        if (t0 < c1) cp_async16(const_cast<uint4*>(sC) + j * kNT + tid, cp_local + (t0 - lo));
        else const_cast<uint4*>(sC)[j * kNT + tid] = make_uint4(0, 0, 0, 0);
      }
      cp_async_commit();
    }
    if (warp == 0) {
      // exclusive scan of the kVPT*kNW warp totals in (j, warp) order; the 16-bit
      // fields do not carry: a chunk holds 32768 tokens
      constexpr int NTOT = kVPT * kNW;
      constexpr int PER = (NTOT + 31) / 32;
      uint32_t loc[PER], s = 0;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int idx = lane * PER + i;
        loc[i] = idx < NTOT ? S.wsum[idx / kNW][idx % kNW] : 0u;
        s += loc[i];
      }
      uint32_t inc = s;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
      }
      uint32_t run = inc - s;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int idx = lane * PER + i;
        if (idx < NTOT) S.wsum[idx / kNW][idx % kNW] = run;
        run += loc[i];
      }
      if (lane == 31) S.wsum_total = run;  // chunk totals
    }
    __syncthreads();
    const uint32_t rgt = S.s_run[0], req = S.s_run[1];
#pragma unroll 1
    for (int j = 0; j < kVPT; ++j) {
      uint32_t p = sPk[j * kNT + tid];
      if (p == 0) continue;
      const uint32_t ex = S.wsum[j][warp] + sIn[j * kNT + tid];
      uint32_t gb = rgt + (ex & 0xffffu), eb = req + (ex >> 16);
      const int t0 = cb + (j * kNT + tid) * 8;
      while (p) {  // selected / tied tokens in increasing token order
        const int e = (__ffs(p) - 1) >> 1;
        const uint32_t c = (p >> (2 * e)) & 3u;
        p &= ~(3u << (2 * e));
        // (positions are < cap by construction; the bound only guards against a
        //  caller-supplied hist that is inconsistent with the codes)
        if (c == 1u) {
          const uint32_t pos = gb + min(eb, m);
          if (pos < cap) selp[pos] = t0 + e;
          ++gb;
        } else {
          if (eb < m && gb + eb < cap) selp[gb + eb] = t0 + e;
          ++eb;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t tot = S.wsum_total;
      S.s_run[0] = rgt + (tot & 0xffffu);
      S.s_run[1] = req + (tot >> 16);
    }
  }
  __syncthreads();
  return S.s_run[0] + min(S.s_run[1], m);
}

template <int MODE>
__device__ __forceinline__ void select_body(const SelArgs& a) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ SelShared S;
  int* cnt = reinterpret_cast<int*>(sm);  // [L]
  uint32_t* key = sm + a.L;               // [L]
  uint32_t* tbl = sm;                     // [W*32], aliases cnt/key once they are dead
  const int tbl_words = max(2 * a.L, a.W * 32);
  uint32_t* sPk = sm + (tbl_words + 3) / 4 * 4;    // [kVPT][kNT] token classes
  uint32_t* sIn = sPk + kVPT * kNT;                // [kVPT][kNT] warp-exclusive counts
  uint4* sC = reinterpret_cast<uint4*>(sIn + kVPT * kNT);  // [kVPT * kNT] one chunk of codes

  const int tid = threadIdx.x;
  const int pair = blockIdx.x;
  const int lo = a.shard_begin, hi = a.shard_begin + a.shard_len;
  const uint16_t* cp_local = a.codes + (size_t)pair * a.n_max;  // local index = global - lo
  const int c0 = max(a.c0, lo), c1 = min(a.c1, hi);             // local part of the candidate range
  A2ATS_PHASE(g_sel_phase, 0);

  if (MODE == kShardHist || MODE == kShardThresh) {
    pdl_wait();
    pdl_trigger();
  }
  if (MODE == kShardHist) {
    load_counts(a, pair, cnt, key, cp_local);
    for (int l = tid; l < a.L; l += kNT) {
      a.cand_out[(size_t)pair * a.L + l] = cnt[l];
      a.cand_keep[(size_t)pair * a.L + l] = cnt[l];
    }
    return;
  }
  if (MODE == kShardThresh) {
    // cnt <- all-reduced histogram; key from agg
    const float* aggp = a.agg + (size_t)pair * a.L;
    for (int l = tid; l < a.L; l += kNT) {
      cnt[l] = a.cand_in[(size_t)pair * a.L + l];
      key[l] = ~ordered_key(__ldg(aggp + l));
    }
    __syncthreads();
    int total = 0;
    for (int l = tid; l < a.L; l += kNT) total += max(cnt[l], 0);
    total = __reduce_add_sync(0xffffffffu, total);
    __shared__ int s_total;
    if (tid == 0) s_total = 0;
    __syncthreads();
    if ((tid & 31) == 0) atomicAdd(&s_total, total);
    __syncthreads();
    const int keff = min(a.keff, s_total);
    uint32_t kstar = 0, m = 0;
    if (keff > 0) {
      radix_kth(a, S, cnt, key, keff);
      kstar = S.s_kstar;
      m = S.s_m;
    }
    // this rank's candidates above / at v*
    int gt = 0, eq = 0;
    if (keff > 0) {
      for (int l = tid; l < a.L; l += kNT) {
        const int c = a.cand_keep[(size_t)pair * a.L + l];
        if (key[l] < kstar) gt += c;
        else if (key[l] == kstar) eq += c;
      }
    }
    gt = __reduce_add_sync(0xffffffffu, gt);
    eq = __reduce_add_sync(0xffffffffu, eq);
    __shared__ int s_gt, s_eq;
    if (tid == 0) s_gt = s_eq = 0;
    __syncthreads();
    if ((tid & 31) == 0) {
      atomicAdd(&s_gt, gt);
      atomicAdd(&s_eq, eq);
    }
    __syncthreads();
    if (tid == 0) {
      a.pinfo[pair * 4 + 0] = kstar;
      a.pinfo[pair * 4 + 1] = m;
      a.pinfo[pair * 4 + 2] = (uint32_t)keff;
      a.counts_out[pair * 2 + 0] = s_gt;
      a.counts_out[pair * 2 + 1] = s_eq;
    }
    return;
  }

  // kFused / kShardScan: prefetch the first chunk of local candidate codes (cp.async -> sC)
  const int first = lo + (((c0 - lo) >> 3) << 3);
  for (int j = 0; j < kVPT; ++j) {
    const int t0 = first + (j * kNT + tid) * 8;
    if (c0 < c1 && t0 < c1) cp_async16(sC + j * kNT + tid, cp_local + (t0 - lo));
    else sC[j * kNT + tid] = make_uint4(0, 0, 0, 0);  // codes past the range must be valid (< L)
  }
  cp_async_commit();
  A2ATS_PHASE(g_sel_phase, 1);
  // the code prefetch above overlaps the predecessor's tail (codes are step inputs)
  pdl_wait();
  pdl_trigger();
  uint32_t kstar, m, cap;
  int32_t* selp;
  if (MODE == kFused) {
    load_counts(a, pair, cnt, key, cp_local);
    A2ATS_PHASE(g_sel_phase, 6);
    radix_kth(a, S, cnt, key, a.keff);
    A2ATS_PHASE(g_sel_phase, 7);
    kstar = S.s_kstar;
    m = S.s_m;
    cap = (uint32_t)a.keff;
    selp = a.sel + (size_t)pair * a.sel_stride;
  } else {
    // shard scan: key from agg, v*/m from shard_thresh, this rank's tie quota from the gather
    const float* aggp = a.agg + (size_t)pair * a.L;
    for (int l = tid; l < a.L; l += kNT) key[l] = ~ordered_key(__ldg(aggp + l));
    kstar = a.pinfo[pair * 4 + 0];
    const int mg = (int)a.pinfo[pair * 4 + 1];
    const int keffg = (int)a.pinfo[pair * 4 + 2];
    int eq_before = 0;
    for (int r = 0; r < a.rank; ++r) eq_before += a.counts_all[((size_t)r * gridDim.x + pair) * 2 + 1];
    const int gt_r = a.counts_all[((size_t)a.rank * gridDim.x + pair) * 2 + 0];
    const int eq_r = a.counts_all[((size_t)a.rank * gridDim.x + pair) * 2 + 1];
    m = keffg > 0 ? (uint32_t)min(max(mg - eq_before, 0), eq_r) : 0u;
    cap = keffg > 0 ? (uint32_t)(gt_r + (int)m) : 0u;
    if (keffg == 0) kstar = 0u;  // nothing above key 0 except impossible keys: emit nothing
    selp = a.sel + (size_t)pair * a.sel_stride;
    if (tid == 0) a.nsel_out[pair] = (int)cap;
    __syncthreads();
  }
  build_table(a, S, key, kstar, tbl);
  A2ATS_PHASE(g_sel_phase, 8);
  if (MODE == kShardScan && cap == 0) return;
  scan_emit(a, S, tbl, cp_local, c0, c1, m, cap, selp, sC, sPk, sIn);
  A2ATS_PHASE(g_sel_phase, 9);
}

template <int MODE>
__global__ __launch_bounds__(kNT, 1) void select_kernel(SelArgs a) {
  A2ATS_TL(g_sel_tl, 0);
  select_body<MODE>(a);
  A2ATS_TL(g_sel_tl, 1);
}

template <int MODE>
cudaError_t launch_mode(const SelArgs& a, int P, cudaStream_t st) {
  const int tbl_words = max(2 * a.L, a.W * 32);
  const int smem = ((tbl_words + 3) / 4 * 4 + 2 * kVPT * kNT) * 4 + kVPT * kNT * 16;
  static int smem_set = -1;
  if (smem_set < smem) {
    cudaError_t e = cudaFuncSetAttribute(select_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  return launch_pdl(select_kernel<MODE>, dim3(P), dim3(kNT), smem, st, a);
}
}  // namespace

cudaError_t launch_select(const SelArgs& a, int P, cudaStream_t st) { return launch_mode<kFused>(a, P, st); }
cudaError_t launch_shard_hist(const SelArgs& a, int P, cudaStream_t st) { return launch_mode<kShardHist>(a, P, st); }
cudaError_t launch_shard_thresh(const SelArgs& a, int P, cudaStream_t st) {
  return launch_mode<kShardThresh>(a, P, st);
}
cudaError_t launch_shard_scan(const SelArgs& a, int P, cudaStream_t st) { return launch_mode<kShardScan>(a, P, st); }

}  // namespace a2ats

A2ATS_PHASE_EXPORT(a2ats_debug_select_phases, a2ats::g_sel_phase)

A2ATS_TL_EXPORT(a2ats_debug_select_timeline, a2ats::g_sel_tl)
