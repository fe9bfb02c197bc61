// a5 + a6: exact softmax attention over Sel = Sinks u TopK u Window
// (Eq. 2) with WRoPE logits (Eq. 11):
//   sinks / top-K rows : u_j = q~ . k_j          (bridge rotation R_b)
//   window rows        : u_j = (q R_{i-j}) . k_j = sum_m cos(r f_m) A_m + sin(r f_m) B_m,
//                        A_m = q_m k_m + q_{m+64} k_{m+64}, B_m = q_m k_{m+64} - q_{m+64} k_m
//                        (the relative identity of Eq. 3 applied to the query only).
// One CTA = one (pair, row split, head subset); 4 warps; each warp takes groups
// of 4 rows, lane = (row-in-group rsub, 16-element slice ds) so that q and the
// output accumulator of GT heads live in registers.  K/V rows are gathered with
// cp.async (16 B per lane-piece) into a warp-private ring of kStages stages; a
// lane consumes exactly the pieces it copied, so the ring needs no barrier.
// fp32 online softmax in base 2; partial (m, l, o) per split; the last CTA of a
// (pair, head subset) combines the splits in fixed order (deterministic LSE).
#include "internal.cuh"

namespace a2ats {

namespace {
constexpr int kStages = 8;
constexpr int kWarps = 4;

struct SmemLayout {
  int tok_off, ring_off, red_off, total;
};
__host__ __device__ inline SmemLayout attn_smem(int R, int GT) {
  SmemLayout s;
  s.tok_off = 0;
  s.ring_off = ((R * 4) + 127) / 128 * 128;
  s.red_off = s.ring_off + kWarps * kStages * 4 * 32 * 16;
  s.total = s.red_off + kWarps * GT * 130 * 4;
  return s;
}

template <int GT>
__global__ __launch_bounds__(128, 2) void sparse_attention_kernel(AttnArgs a) {
  extern __shared__ __align__(128) uint8_t smraw[];
  const SmemLayout L = attn_smem(a.R, GT);
  int32_t* s_tok = reinterpret_cast<int32_t*>(smraw + L.tok_off);
  uint4* ring = reinterpret_cast<uint4*>(smraw + L.ring_off);
  float* red = reinterpret_cast<float*>(smraw + L.red_off);

  const int split = blockIdx.x, pair = blockIdx.y, gz = blockIdx.z;
  const int nz = gridDim.z;
  const int b = pair / a.Hkv, h = pair - (pair / a.Hkv) * a.Hkv;
  const int hq0 = h * a.G + gz * GT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, rsub = lane >> 3, ds = lane & 7;

  const int p0 = split * a.R;
  const int p1 = min(p0 + a.R, a.M);
  const int pw = a.n_s + a.keff;  // first window position in the Sel list
  // segment A (bridge rows) and segment B (window rows) of this split
  const int nA = max(0, min(p1, pw) - p0);
  const int nB = (p1 - p0) - nA;
  const int gA = (nA + 3) >> 2, gB = (nB + 3) >> 2;
  const int ngroups = gA + gB;

  for (int i = tid; i < p1 - p0; i += 128) {
    const int p = p0 + i;
    int t;
    if (p < a.n_s) t = p;
    else if (p < pw) t = a.sel[(size_t)pair * a.keff + (p - a.n_s)];
    else t = a.w0 + (p - pw);
    s_tok[i] = t;
  }
  __syncthreads();

  const size_t rowbase = (size_t)pair * a.n_max;
  const uint8_t* kbase = reinterpret_cast<const uint8_t*>(a.kc) + rowbase * 256;
  const uint8_t* vbase = reinterpret_cast<const uint8_t*>(a.vc) + rowbase * 256;
  uint4* wring = ring + warp * (kStages * 4 * 32);

  auto local_row = [&](int g, int& li) -> bool {
    if (g < gA) {
      li = g * 4 + rsub;
      return li < nA;
    }
    li = nA + (g - gA) * 4 + rsub;
    return li < nA + nB;
  };
  auto issue = [&](int s) {
    const int g = s * kWarps + warp;
    int li;
    if (g < ngroups && local_row(g, li)) {
      const size_t off = (size_t)s_tok[li] * 256 + ds * 16;
      uint4* slot = wring + (s % kStages) * (4 * 32);
      cp_async16(slot + 0 * 32 + lane, kbase + off);
      cp_async16(slot + 1 * 32 + lane, kbase + off + 128);
      cp_async16(slot + 2 * 32 + lane, vbase + off);
      cp_async16(slot + 3 * 32 + lane, vbase + off + 128);
    }
    cp_async_commit();
  };

  // q~ (bridge), pre-scaled by log2(e)/sqrt(d): lane holds elements ds*8+i and 64+ds*8+i.
  float qr[GT][16];
#pragma unroll
  for (int g = 0; g < GT; ++g) {
    const float* src = a.qrot + ((size_t)b * a.Hq + hq0 + g) * kD;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      qr[g][i] = src[ds * 8 + i] * a.scale_log2;
      qr[g][8 + i] = src[kHalf + ds * 8 + i] * a.scale_log2;
    }
  }
  float o[GT][16], mrun[GT], lsum[GT];
#pragma unroll
  for (int g = 0; g < GT; ++g) {
    mrun[g] = -INFINITY;
    lsum[g] = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) o[g][i] = 0.f;
  }

  const int nsteps = (ngroups > warp) ? (ngroups - warp + kWarps - 1) / kWarps : 0;
#pragma unroll 1
  for (int s = 0; s < kStages - 1; ++s) issue(s);

  bool in_window = false;
  const int icur = a.n_ctx - 1;
#pragma unroll 1
  for (int s = 0; s < nsteps; ++s) {
    issue(s + kStages - 1);
    cp_async_wait<kStages - 1>();
    const int g = s * kWarps + warp;
    int li;
    const bool valid = local_row(g, li);
    const bool win = g >= gA;
    if (win && !in_window) {
      // switch the query registers to the raw (pre-PE) query for the window band
#pragma unroll
      for (int gg = 0; gg < GT; ++gg) {
        const uint16_t* src = a.q + ((size_t)b * a.Hq + hq0 + gg) * kD;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          qr[gg][i] = bf_u16(src[ds * 8 + i]) * a.scale_log2;
          qr[gg][8 + i] = bf_u16(src[kHalf + ds * 8 + i]) * a.scale_log2;
        }
      }
      in_window = true;
    }
    const uint4* slot = wring + (s % kStages) * (4 * 32);
    const uint4 k0 = slot[0 * 32 + lane], k1 = slot[1 * 32 + lane];
    float kf[16];
    {
      const uint32_t w[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        kf[2 * i] = bf_lo(w[i]);
        kf[2 * i + 1] = bf_hi(w[i]);
      }
    }
    float sc[GT];
    if (!win) {
#pragma unroll
      for (int gg = 0; gg < GT; ++gg) {
        float x = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) x = fmaf(qr[gg][i], kf[i], x);
        sc[gg] = x;
      }
    } else {
      const int r = valid ? (icur - s_tok[li]) : 0;
      const float4* csp = reinterpret_cast<const float4*>(a.cs + (size_t)r * kHalf + ds * 8);
      float cv[8], sv[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 t = csp[i];
        cv[2 * i] = t.x; sv[2 * i] = t.y; cv[2 * i + 1] = t.z; sv[2 * i + 1] = t.w;
      }
#pragma unroll
      for (int gg = 0; gg < GT; ++gg) {
        float x = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float A = fmaf(qr[gg][i], kf[i], qr[gg][8 + i] * kf[8 + i]);
          const float Bm = fmaf(qr[gg][i], kf[8 + i], -qr[gg][8 + i] * kf[i]);
          x = fmaf(cv[i], A, fmaf(sv[i], Bm, x));
        }
        sc[gg] = x;
      }
    }
#pragma unroll
    for (int gg = 0; gg < GT; ++gg) {
      sc[gg] += __shfl_xor_sync(0xffffffffu, sc[gg], 1);
      sc[gg] += __shfl_xor_sync(0xffffffffu, sc[gg], 2);
      sc[gg] += __shfl_xor_sync(0xffffffffu, sc[gg], 4);
    }
    if (valid) {
      const uint4 v0 = slot[2 * 32 + lane], v1 = slot[3 * 32 + lane];
      const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      float vf[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        vf[2 * i] = bf_lo(w[i]);
        vf[2 * i + 1] = bf_hi(w[i]);
      }
#pragma unroll
      for (int gg = 0; gg < GT; ++gg) {
        if (sc[gg] > mrun[gg]) {
          const float corr = exp2f(mrun[gg] - sc[gg]);
          lsum[gg] *= corr;
#pragma unroll
          for (int i = 0; i < 16; ++i) o[gg][i] *= corr;
          mrun[gg] = sc[gg];
        }
        const float p = exp2f(sc[gg] - mrun[gg]);
        lsum[gg] += p;
#pragma unroll
        for (int i = 0; i < 16; ++i) o[gg][i] = fmaf(p, vf[i], o[gg][i]);
      }
    }
  }
  cp_async_wait<0>();

  // combine the 4 row-slots (rsub) of the warp: lanes ds, ds+8, ds+16, ds+24
#pragma unroll
  for (int gg = 0; gg < GT; ++gg) {
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, mrun[gg], off);
      const float lo = __shfl_xor_sync(0xffffffffu, lsum[gg], off);
      const float mn = fmaxf(mrun[gg], mo);
      const float a1 = (mrun[gg] == -INFINITY) ? 0.f : exp2f(mrun[gg] - mn);
      const float a2 = (mo == -INFINITY) ? 0.f : exp2f(mo - mn);
      lsum[gg] = lsum[gg] * a1 + lo * a2;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float oo = __shfl_xor_sync(0xffffffffu, o[gg][i], off);
        o[gg][i] = o[gg][i] * a1 + oo * a2;
      }
      mrun[gg] = mn;
    }
  }
  // element index of o[gg][i]: i < 8 -> ds*8+i, else 64 + ds*8 + (i-8)
  if (rsub == 0) {
#pragma unroll
    for (int gg = 0; gg < GT; ++gg) {
      float* r = red + (warp * GT + gg) * 130;
      if (ds == 0) {
        r[0] = mrun[gg];
        r[1] = lsum[gg];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        r[2 + ds * 8 + i] = o[gg][i];
        r[2 + kHalf + ds * 8 + i] = o[gg][8 + i];
      }
    }
  }
  __syncthreads();

  // combine the 4 warps: thread tid -> element e = tid (128 threads = d)
  const int e = tid;
  const int pz = pair * nz + gz;
  float* part = a.part + (size_t)pz * GT * a.nsplit * 130;
  const bool single = (a.nsplit == 1);
#pragma unroll
  for (int gg = 0; gg < GT; ++gg) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, red[(w * GT + gg) * 130]);
    float acc = 0.f, den = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float mw = red[(w * GT + gg) * 130];
      const float sw = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      acc = fmaf(red[(w * GT + gg) * 130 + 2 + e], sw, acc);
      den = fmaf(red[(w * GT + gg) * 130 + 1], sw, den);
    }
    if (single) {
      a.out[((size_t)b * a.Hq + hq0 + gg) * kD + e] = acc / den;
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
    const unsigned prev = atomicAdd(a.counter + pz, 1u);
    s_last = (prev == (unsigned)(a.nsplit - 1));
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
#pragma unroll 1
  for (int gg = 0; gg < GT; ++gg) {
    const float* src = part + (size_t)gg * a.nsplit * 130;
    float M = -INFINITY;
    for (int s = 0; s < a.nsplit; ++s) M = fmaxf(M, __ldcg(src + s * 130));
    float num = 0.f, den = 0.f;
    for (int s = 0; s < a.nsplit; ++s) {
      const float ms = __ldcg(src + s * 130);
      const float sw = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
      num = fmaf(__ldcg(src + s * 130 + 2 + e), sw, num);
      den = fmaf(__ldcg(src + s * 130 + 1), sw, den);
    }
    a.out[((size_t)b * a.Hq + hq0 + gg) * kD + e] = num / den;
  }
  if (tid == 0) a.counter[pz] = 0u;  // leave the workspace in its zero state
}

template <int GT>
cudaError_t launch_attn_t(const AttnArgs& a, int P, cudaStream_t st) {
  const SmemLayout L = attn_smem(a.R, GT);
  static int smem_set = -1;
  if (smem_set < L.total) {
    cudaError_t e = cudaFuncSetAttribute(sparse_attention_kernel<GT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         L.total);
    if (e != cudaSuccess) return e;
    smem_set = L.total;
  }
  dim3 grid(a.nsplit, P, a.G / GT);
  sparse_attention_kernel<GT><<<grid, 128, L.total, st>>>(a);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_attention(const AttnArgs& a, int P, int GT, cudaStream_t st) {
  switch (GT) {
    case 1: return launch_attn_t<1>(a, P, st);
    case 2: return launch_attn_t<2>(a, P, st);
    default: return launch_attn_t<4>(a, P, st);
  }
}

}  // namespace a2ats
