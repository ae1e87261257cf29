// The per-block x-window in shared memory: x[wlo, wlo + W) staged with
// coalesced loads into a padded layout (16-entry tiles at a stride of 17
// entries, so a thread can walk one tile with 2-way bank conflicts), plus a
// tile-local exclusive prefix in double-double (hi fp64, lo fp32) and the
// tile totals.  An interval [a, e) spanning at most two tiles is then
//     (e tile != a tile ? T[a tile] : 0) - P[a] + P[e]
// evaluated with two TwoSums -- O(1), branch-free, and accurate to ~1e-30
// absolute, so interval sums carry no rounding error into the reference
// chain (the north star's O(1) interval evaluation from an exclusive prefix).
#pragma once
#include <cstdint>

namespace cmvg {

__host__ __device__ constexpr uint32_t xw_pad(uint32_t j) { return j + (j >> 4); }

// bytes of the x-window region for W entries of type XT
__host__ __device__ inline uint32_t xw_bytes(uint32_t W, uint32_t xsize, bool prefix) {
  const uint32_t padded = xw_pad(W) + 1;
  uint32_t b = ((padded * xsize + 15u) & ~15u);
  if (prefix) {
    b += ((padded * 8u + 15u) & ~15u);          // P hi
    b += ((padded * 4u + 15u) & ~15u);          // P lo
    b += (((W / 16 + 1) * 8u + 15u) & ~15u);    // T hi
    b += (((W / 16 + 1) * 4u + 15u) & ~15u);    // T lo
  }
  return b;
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

template <typename XT, bool PREFIX>
struct XWin {
  XT* s_x;
  double* s_ph;
  float* s_pl;
  double* s_th;
  float* s_tl;
  const XT* __restrict__ x;
  uint32_t wlo, W;

  __device__ __forceinline__ void carve(unsigned char* base, uint32_t Wn) {
    W = Wn;
    const uint32_t padded = xw_pad(Wn) + 1;
    unsigned char* p = base;
    s_x = reinterpret_cast<XT*>(p);
    p += (padded * sizeof(XT) + 15u) & ~15u;
    s_ph = reinterpret_cast<double*>(p);
    p += (padded * 8u + 15u) & ~15u;
    s_pl = reinterpret_cast<float*>(p);
    p += (padded * 4u + 15u) & ~15u;
    s_th = reinterpret_cast<double*>(p);
    p += ((Wn / 16 + 1) * 8u + 15u) & ~15u;
    s_tl = reinterpret_cast<float*>(p);
  }

  // Cooperative staging (all threads of the CTA); ends with __syncthreads().
  __device__ __forceinline__ void stage(uint32_t n) {
    const uint32_t T = blockDim.x, tid = threadIdx.x;
    for (uint32_t j = tid; j < W; j += T) {
      const uint32_t c = wlo + j;
      s_x[xw_pad(j)] = c < n ? __ldg(x + c) : XT(0);
    }
    if constexpr (PREFIX) {
      __syncthreads();
      const uint32_t ntiles = W >> 4;
      for (uint32_t t = tid; t < ntiles; t += T) {
        const uint32_t base = t * 17u;
        double hi = 0.0, lo = 0.0;
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j) {
          s_ph[base + j] = hi;
          s_pl[base + j] = (float)lo;
          double s, e;
          two_sum(hi, (double)s_x[base + j], s, e);
          hi = s;
          lo += e;
        }
        // renormalise the total
        const double h2 = hi + lo;
        s_th[t] = h2;
        s_tl[t] = (float)(lo - (h2 - hi));
      }
    }
    __syncthreads();
  }

  __device__ __forceinline__ double at(int32_t c) const {
    const uint32_t j = (uint32_t)(c - (int32_t)wlo);
    const bool in = j < W;
    XT v = s_x[xw_pad(in ? j : 0u)];
    if (!in) v = __ldg(x + c);  // rare: column outside the window
    return (double)v;
  }

  // sum of x[left, left+len) as (hi, lo)
  __device__ __forceinline__ double isum(int32_t left, uint32_t len, double& lo) const {
    const uint32_t a = (uint32_t)(left - (int32_t)wlo);
    const uint32_t e = a + len;
    if constexpr (PREFIX) {
      const uint32_t ta = a >> 4, tb = e >> 4;
      if (a < W && e <= W && tb <= ta + 1) {
        const bool two = tb != ta;
        const bool has_e = (e & 15u) != 0;
        const uint32_t pa = xw_pad(a), pe = xw_pad(e);
        const double th = two ? s_th[ta] : 0.0;
        const float tl = two ? s_tl[ta] : 0.0f;
        const double peh = has_e ? s_ph[pe] : 0.0;
        const float pel = has_e ? s_pl[pe] : 0.0f;
        double s1, e1, s2, e2;
        two_sum(th, -s_ph[pa], s1, e1);
        two_sum(s1, peh, s2, e2);
        lo = e1 + e2 + ((double)tl - (double)s_pl[pa] + (double)pel);
        return s2;
      }
    } else {
      if (a < W && e <= W && len <= 32) {
        double s = 0.0, c = 0.0;
        for (uint32_t t = a; t < e; ++t) {
          double u, er;
          two_sum(s, (double)s_x[xw_pad(t)], u, er);
          s = u;
          c += er;
        }
        lo = c;
        return s;
      }
    }
    // long or out-of-window interval: compensated sum from global memory
    double s = 0.0, c = 0.0;
    for (uint32_t t = 0; t < len; ++t) {
      double u, er;
      two_sum(s, (double)__ldg(x + left + t), u, er);
      s = u;
      c += er;
    }
    lo = c;
    return s;
  }
};

}  // namespace cmvg
