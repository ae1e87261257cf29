// The per-block x-window in shared memory: x[wlo, wlo + W) staged with
// coalesced loads into a padded layout (8-entry tiles at a stride of 9
// entries, so a thread walks one tile with at most 2-way bank conflicts), plus
// an exclusive prefix F of the window in double-double (hi fp64, lo fp32),
// built in three parallel steps: the 8-entry tile totals (one thread per
// tile), their exclusive prefix Q (one warp), then F within each tile
// starting from Q (one thread per tile) -- x is read twice and F written
// once.  An interval [a, e) is then F[e] - F[a]: one TwoSum, O(1) for any
// length, and accurate to ~1e-28 absolute, so interval sums carry no rounding
// error into the reference chain (the north star's O(1) interval evaluation
// from an exclusive prefix of x).
#pragma once
#include <cstdint>

#include "../host/layout.hpp"

namespace cmvg {

constexpr uint32_t kXwTile = 8;  // entries per tile (bvs_pad_index: stride 9)
__host__ __device__ constexpr uint32_t xw_pad(uint32_t j) { return bvs_pad_index(j); }

// bytes of the x-window region for W entries of type XT (x, F hi / lo, Q hi / lo)
__host__ __device__ inline uint32_t xw_bytes(uint32_t W, uint32_t xsize) {
  const uint32_t padded = xw_pad(W) + 1;
  uint32_t b = ((padded * xsize + 15u) & ~15u);
  b += ((padded * 8u + 15u) & ~15u);                // F hi
  b += ((padded * 4u + 15u) & ~15u);                // F lo
  b += (((W / kXwTile + 1) * 8u + 15u) & ~15u);    // Q hi
  b += (((W / kXwTile + 1) * 4u + 15u) & ~15u);    // Q lo
  return b;
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

template <typename XT>
struct XWin {
  XT* s_x;
  double* s_ph;
  float* s_pl;
  double* s_th;
  float* s_tl;
  const XT* __restrict__ x;
  const XT* xfar;  // x at the columns outside the window (only those are read from it)
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
    p += ((Wn / kXwTile + 1) * 8u + 15u) & ~15u;
    s_tl = reinterpret_cast<float*>(p);
  }

  // Register prefetch of the first kPre*T window entries: issued before the
  // stream wait and row setup so the global-load latency overlaps them.
  static constexpr uint32_t kPre = 8;
  __device__ __forceinline__ void prefetch(uint32_t n, XT (&r)[kPre]) const {
#pragma unroll
    for (uint32_t q = 0; q < kPre; ++q) {
      const uint32_t j = threadIdx.x + q * blockDim.x, c = wlo + j;
      r[q] = (j < W && c < n) ? __ldg(x + c) : XT(0);
    }
  }

  // Cooperative staging (all threads of the CTA); ends with __syncthreads().
  __device__ __forceinline__ void stage(uint32_t n) {
    XT r[kPre];
    prefetch(n, r);
    stage(n, r);
  }
  __device__ __forceinline__ void stage(uint32_t n, const XT (&r)[kPre]) {
    const uint32_t T = blockDim.x, tid = threadIdx.x;
#pragma unroll
    for (uint32_t q = 0; q < kPre; ++q) {
      const uint32_t j = tid + q * T;
      if (j < W) s_x[xw_pad(j)] = r[q];
    }
    if (tid == 0) s_x[xw_pad(W)] = XT(0);  // zero entry for idle lanes
    for (uint32_t j = tid + kPre * T; j < W; j += T) {
      const uint32_t c = wlo + j;
      s_x[xw_pad(j)] = c < n ? __ldg(x + c) : XT(0);
    }
    {
      __syncthreads();
      const uint32_t ntiles = W / kXwTile;
      for (uint32_t t = tid; t < ntiles; t += T) {  // tile totals
        const uint32_t base = t * (kXwTile + 1);
        double hi = 0.0, lo = 0.0;
#pragma unroll
        for (uint32_t j = 0; j < kXwTile; ++j) {
          double s, e;
          two_sum(hi, (double)s_x[base + j], s, e);
          hi = s;
          lo += e;
        }
        const double h2 = hi + lo;
        s_th[t] = h2;
        s_tl[t] = (float)(lo - (h2 - hi));
      }
      __syncthreads();
      if (tid < 32) {  // Q: exclusive double-double prefix of the tile totals (one warp)
        const uint32_t lane = tid, per = (ntiles + 31u) / 32u;
        double lh = 0.0, ll = 0.0;
        for (uint32_t q = 0; q < per; ++q) {
          const uint32_t t = lane * per + q;
          if (t < ntiles) {
            double s, e;
            two_sum(lh, s_th[t], s, e);
            lh = s;
            ll += e + (double)s_tl[t];
          }
        }
        double ih = lh, il = ll;  // inclusive warp scan in double-double
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double uh = __shfl_up_sync(0xffffffffu, ih, o), ul = __shfl_up_sync(0xffffffffu, il, o);
          if ((int)lane >= o) {
            double s, e;
            two_sum(ih, uh, s, e);
            ih = s;
            il += ul + e;
          }
        }
        double rh = __shfl_up_sync(0xffffffffu, ih, 1), rl = __shfl_up_sync(0xffffffffu, il, 1);
        if (lane == 0) rh = rl = 0.0;
        for (uint32_t q = 0; q < per; ++q) {
          const uint32_t t = lane * per + q;
          if (t < ntiles) {
            const double th = s_th[t];
            const float tl = s_tl[t];
            const double h2 = rh + rl;
            s_th[t] = h2;  // in place: tile total -> exclusive prefix Q[t]
            s_tl[t] = (float)(rl - (h2 - rh));
            double s, e;
            two_sum(rh, th, s, e);
            rh = s;
            rl += e + (double)tl;
          }
        }
        if (lane == 31) {
          const double h2 = ih + il;
          s_th[ntiles] = h2;
          s_tl[ntiles] = (float)(il - (h2 - ih));
        }
      }
      __syncthreads();
      for (uint32_t t = tid; t < ntiles; t += T) {  // F within each tile, from Q[t]
        const uint32_t base = t * (kXwTile + 1);
        double hi = s_th[t], lo = (double)s_tl[t];
#pragma unroll
        for (uint32_t j = 0; j < kXwTile; ++j) {
          const double h2 = hi + lo;
          s_ph[base + j] = h2;
          s_pl[base + j] = (float)(lo - (h2 - hi));
          double s, e;
          two_sum(hi, (double)s_x[base + j], s, e);
          hi = s;
          lo += e;
        }
      }
      if (tid == 0) {  // F at the window end: the total
        s_ph[xw_pad(W)] = s_th[ntiles];
        s_pl[xw_pad(W)] = s_tl[ntiles];
      }
    }
    __syncthreads();
  }

  // Unchecked accessors for `near` rows (the builder guarantees the window
  // holds every column): j, a are window-relative, p a padded index.
  __device__ __forceinline__ double at_near(uint32_t j) const { return (double)s_x[xw_pad(j)]; }
  __device__ __forceinline__ double at_padded(uint32_t p) const { return (double)s_x[p]; }
  __device__ __forceinline__ double isum_near(uint32_t a, uint32_t len, double& lo) const {
    const uint32_t pa = xw_pad(a), pe = xw_pad(a + len);
    double s, e;
    two_sum(s_ph[pe], -s_ph[pa], s, e);
    lo = e + ((double)s_pl[pe] - (double)s_pl[pa]);
    return s;
  }

  __device__ __forceinline__ double at(int32_t c) const {
    const uint32_t j = (uint32_t)(c - (int32_t)wlo);
    const bool in = j < W;
    XT v = s_x[xw_pad(in ? j : 0u)];
    if (!in) v = __ldg(xfar + c);  // rare: column outside the window (read-only during the kernel)
    return (double)v;
  }

  // sum of x[left, left+len) as (hi, lo): O(1) from the prefix inside the
  // window, otherwise a compensated sum entry by entry (window entries from
  // shared memory, the others from xfar: xfar need only hold the columns
  // outside the window)
  __device__ __forceinline__ double isum(int32_t left, uint32_t len, double& lo) const {
    const uint32_t a = (uint32_t)(left - (int32_t)wlo);
    if (a < W && a + len <= W) return isum_near(a, len, lo);
    double s = 0.0, c = 0.0;
    for (uint32_t t = 0; t < len; ++t) {
      double u, er;
      two_sum(s, at(left + (int32_t)t), u, er);  // a run may straddle the window edge
      s = u;
      c += er;
    }
    lo = c;
    return s;
  }
};

}  // namespace cmvg
