// a3 + a4: approximate scores through the code stream and exact top-K selection.
//
// Scores take only L distinct values per (b, KV head) pair (u^_t = LUT[s_t],
// Eq. 21), so the K-th largest score is found by a count-weighted
// radix select over the L codewords, not over the N tokens.  One CTA owns one
// pair (fused kernel, no intermediate in HBM):
//
//  1. issue the 128-bit loads of the first code chunk (registers), so the DRAM
//     latency overlaps steps 2-4;
//  2. candidate histogram over codewords: the caller-maintained hist minus the
//     sink/window codes (one pass over the code stream in total), or, without
//     hist, an extra pass over the codes;
//  3. count-weighted MSB-first radix select of the K-th largest agg level v*
//     (warp-aggregated shared atomics: float keys share their top bits);
//     tie quota m = K - #{agg > v*};
//  4. 2-bit class per codeword (1: agg > v*, 2: agg == v*), replicated 32x in
//     shared memory so lane l reads bank l (conflict-free gather by code);
//  5. stream the codes chunk by chunk (next chunk prefetched into registers),
//     classify each token, and write the selected indices in ascending order
//     (block scan + running prefix).  A token with agg == v* is kept iff fewer
//     than m such tokens precede it: the lowest-index tie-break of reading Q12.
#include "internal.cuh"

namespace a2ats {

namespace {

__device__ __forceinline__ uint32_t spread16(uint32_t v) {
  v &= 0xffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}


template <int NT, int VPT>
__global__ __launch_bounds__(NT, 1) void select_fused_kernel(SelArgs a) {
  constexpr int NW = NT / 32;
  constexpr int CH = NT * VPT * 8;  // tokens per chunk
  extern __shared__ __align__(16) uint32_t sm[];
  int* cnt = reinterpret_cast<int*>(sm);  // [L]
  uint32_t* key = sm + a.L;               // [L] ~ordered(agg): ascending key = descending agg
  uint32_t* tbl = sm;                     // [W*32] aliases cnt/key after step 4
  __shared__ uint32_t cls[1024];          // compact 2-bit classes (W <= 1024)
  __shared__ int bins[256];
  __shared__ int whist[NW * 256];         // per-warp digit histograms
  __shared__ uint32_t wsum[VPT][NW];
  __shared__ int s_digit, s_kk;
  __shared__ uint32_t s_run[2];
  __shared__ uint32_t s_and, s_or;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x;
  const uint16_t* cp = a.codes + (size_t)pair * a.n_max;
  const int c0 = a.c0, c1 = a.c1;
  const int first = (c0 >> 3) << 3;                   // 8-aligned start of the candidate range
  const int nchunk = (c1 - first + CH - 1) / CH;

  // 1. prefetch chunk 0
  uint4 v[VPT];
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int t0 = first + (j * NT + tid) * 8;
    v[j] = (t0 < c1) ? ld_stream_u4(cp + t0) : make_uint4(0, 0, 0, 0);
  }

  // 2. candidate histogram
  if (tid == 0) {
    s_and = 0xffffffffu;
    s_or = 0u;
  }
  const float* aggp = a.agg + (size_t)pair * a.L;
  for (int l = tid; l < a.L; l += NT) {
    cnt[l] = a.hist ? a.hist[(size_t)pair * a.L + l] : 0;
    key[l] = ~ordered_key(aggp[l]);
  }
  __syncthreads();
  if (a.hist) {
    const int nrem = a.n_s + (a.n_ctx - a.w0);
    for (int i = tid; i < nrem; i += NT) {
      const int t = i < a.n_s ? i : a.w0 + (i - a.n_s);
      atomicSub(&cnt[cp[t]], 1);
    }
  } else {
    for (int vi = (first >> 3) + tid; vi < ((c1 + 7) >> 3); vi += NT) {
      const uint4 x = ld_nc_u4(cp + (size_t)vi * 8);
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int t = vi * 8 + e;
        if (t >= c0 && t < c1) atomicAdd(&cnt[(w[e >> 1] >> ((e & 1) * 16)) & 0xffffu], 1);
      }
    }
  }
  __syncthreads();

  // 3. radix select of the keff-th smallest key, weighted by counts.  Bits common to
  //    every candidate key are skipped; digits are counted in per-warp histograms.
  uint32_t kand = 0xffffffffu, kor = 0u;
  for (int l = tid; l < a.L; l += NT) {
    if (cnt[l] > 0) {
      kand &= key[l];
      kor |= key[l];
    }
  }
  kand = __reduce_and_sync(0xffffffffu, kand);
  kor = __reduce_or_sync(0xffffffffu, kor);
  if (lane == 0) {
    atomicAnd(&s_and, kand);
    atomicOr(&s_or, kor);
  }
  __syncthreads();
  const uint32_t diff = s_and ^ s_or;            // bits where candidate keys differ
  const int top = diff ? 31 - __clz(diff) : 0;   // highest differing bit
  const int npass = diff ? (top / 8) + 1 : 0;    // passes over digits [8*(npass-1), ...]
  uint32_t prefix = diff ? (s_and & ~((top >= 31) ? 0xffffffffu : ((2u << top) - 1u))) : s_and;
  uint32_t mask = diff ? ~((top >= 31) ? 0xffffffffu : ((2u << top) - 1u)) : 0xffffffffu;
  int kk = a.keff;
  for (int pass = npass - 1; pass >= 0; --pass) {
    const int shift = 8 * pass;
    for (int i = tid; i < NW * 256; i += NT) whist[i] = 0;
    __syncthreads();
    int* wh = whist + warp * 256;
    for (int l = tid; l < a.L; l += NT) {
      const int c = cnt[l];
      const uint32_t k = key[l];
      if (c > 0 && (k & mask) == prefix) atomicAdd(wh + ((k >> shift) & 255u), c);
    }
    __syncthreads();
    for (int i = tid; i < 256; i += NT) {
      int s = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += whist[w * 256 + i];
      bins[i] = s;
    }
    __syncthreads();
    if (warp == 0) {
      int loc[8], s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        loc[i] = bins[lane * 8 + i];
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
            s_digit = lane * 8 + i;
            s_kk = kk - c;
            break;
          }
          c += loc[i];
        }
      }
    }
    __syncthreads();
    // digit bits above `top` are part of the common prefix already; OR-ing is idempotent
    prefix = (prefix & ~(0xffu << shift)) | ((uint32_t)s_digit << shift);
    mask |= 0xffu << shift;
    kk = s_kk;
  }
  const uint32_t kstar = prefix;  // key of v*;  kk = tie quota m >= 1
  const uint32_t m = (uint32_t)kk;

  // 4. classes: compact words, then 32x replication over the (dead) cnt/key arrays
  for (int gi = warp; gi < (a.L + 31) / 32; gi += NW) {
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
      cls[gi * 2 + lane] = spread16(g16) | (spread16(e16) << 1);
    }
  }
  if (tid == 0) {
    s_run[0] = 0;
    s_run[1] = 0;
  }
  __syncthreads();
  for (int i = tid; i < a.W * 32; i += NT) tbl[i] = cls[i >> 5];
  __syncthreads();

  // 5. classify + ordered compaction, chunk by chunk
  int32_t* selp = a.sel + (size_t)pair * a.keff;
  const uint32_t keff = (uint32_t)a.keff;
  for (int ch = 0; ch < nchunk; ++ch) {
    const int cb = first + ch * CH;
    uint32_t packed[VPT], pk[VPT], incl[VPT];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int t0 = cb + (j * NT + tid) * 8;
      const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
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
      packed[j] = p;
    }
    // prefetch the next chunk while this one is scanned
    if (ch + 1 < nchunk) {
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const int t0 = cb + CH + (j * NT + tid) * 8;
        v[j] = (t0 < c1) ? ld_stream_u4(cp + t0) : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      pk[j] = (uint32_t)__popc(packed[j] & 0x5555u) | ((uint32_t)__popc(packed[j] & 0xaaaau) << 16);
      uint32_t x = pk[j];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      incl[j] = x;
      if (lane == 31) wsum[j][warp] = x;
    }
    __syncthreads();
    if (warp == 0) {
      // exclusive scan of the VPT*NW warp totals in (j, warp) order; 16-bit fields
      // do not carry: a chunk holds <= 65535 tokens.
      constexpr int NTOT = VPT * NW;
      constexpr int PER = (NTOT + 31) / 32;
      uint32_t loc[PER], s = 0;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int idx = lane * PER + i;
        loc[i] = idx < NTOT ? wsum[idx / NW][idx % NW] : 0u;
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
        if (idx < NTOT) wsum[idx / NW][idx % NW] = run;
        run += loc[i];
      }
    }
    __syncthreads();
    const uint32_t rgt = s_run[0], req = s_run[1];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const uint32_t p = packed[j];
      if (p == 0) continue;
      const uint32_t ex = wsum[j][warp] + incl[j] - pk[j];
      uint32_t gb = rgt + (ex & 0xffffu), eb = req + (ex >> 16);
      const int t0 = cb + (j * NT + tid) * 8;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t c = (p >> (2 * e)) & 3u;
        // (positions are < keff by construction; the bound only guards against a
        //  caller-supplied hist that is inconsistent with the codes)
        if (c == 1u) {
          const uint32_t pos = gb + min(eb, m);
          if (pos < keff) selp[pos] = t0 + e;
          ++gb;
        } else if (c == 2u) {
          if (eb < m && gb + eb < keff) selp[gb + eb] = t0 + e;
          ++eb;
        }
      }
    }
    __syncthreads();
    if (tid == NT - 1) {
      // chunk totals = last (j, warp) exclusive prefix + its own count
      const uint32_t tot = wsum[VPT - 1][NW - 1] + incl[VPT - 1];
      s_run[0] = rgt + (tot & 0xffffu);
      s_run[1] = req + (tot >> 16);
    }
    __syncthreads();
  }
}

template <int NT, int VPT>
cudaError_t launch_fused(const SelArgs& a, int P, cudaStream_t st) {
  const int smem = max(a.L * 8, a.W * 32 * 4);
  static int smem_set = -1;
  if (smem_set < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(select_fused_kernel<NT, VPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  select_fused_kernel<NT, VPT><<<P, NT, smem, st>>>(a);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_select(const SelArgs& a, int P, cudaStream_t st) {
  // one CTA per pair; 512 threads x 8 x 128-bit loads = 32768 tokens per chunk
  return launch_fused<512, 8>(a, P, st);
}

}  // namespace a2ats
