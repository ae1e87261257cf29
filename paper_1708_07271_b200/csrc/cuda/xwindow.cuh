// The per-block x-window in shared memory: x[wlo, wlo + W) in a padded layout
// (8-entry tiles at a stride of 9 entries; the transcoder's codes are padded
// indices), plus an exclusive prefix F of the window in double-double (hi
// fp64, lo fp32).  Staging is one pass per round of T x E entries (E <= 8
// contiguous entries per thread, E = W / T = 6 at the default W = 1536,
// T = 256): each thread loads its chunk with paired (16-B) loads issued before
// the CTA's first barrier, sums it in double-double, the chunk totals are
// scanned with warp shuffles and one barrier for the warp totals, and each
// thread then writes its x entries and their prefix values F from registers.
// An interval [a, e) is then F[e] - F[a]: one TwoSum, O(1) for any length,
// and accurate to ~1e-28 absolute, so interval sums carry no rounding error
// into the reference chain (the north star's O(1) interval evaluation from an
// exclusive prefix of x).
#pragma once
#include <cstdint>
#include <type_traits>

#include "../host/layout.hpp"

namespace cmvg {

constexpr uint32_t kXwTile = 8;  // entries per tile (bvs_pad_index: stride 9)
__host__ __device__ constexpr uint32_t xw_pad(uint32_t j) { return bvs_pad_index(j); }

// warp-total scratch of the staging scan (2 doubles per warp, <= 32 warps, + carry)
constexpr uint32_t kXwScratch = 2 * 32 + 2;

// bytes of the x-window region for W entries of type XT (x, F hi / lo, scratch)
__host__ __device__ inline uint32_t xw_bytes(uint32_t W, uint32_t xsize) {
  const uint32_t padded = xw_pad(W) + 1;
  uint32_t b = ((padded * xsize + 15u) & ~15u);
  b += ((padded * 8u + 15u) & ~15u);  // F hi
  b += ((padded * 4u + 15u) & ~15u);  // F lo
  b += kXwScratch * 8u;               // warp totals
  return b;
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

template <typename XT>
struct XWin {
  using value_type = XT;
  XT* s_x;
  double* s_ph;
  float* s_pl;
  double* s_wt;  // staging scratch: warp totals, carry
  const XT* __restrict__ x;
  const XT* xfar;  // x at the columns outside the window (only those are read from it)
  uint32_t wlo, W;
  uint32_t T;  // threads of the CTA (a power of two; a compile-time constant in the specialised kernels)

  __device__ __forceinline__ void carve(unsigned char* base, uint32_t Wn, uint32_t threads) {
    W = Wn;
    T = threads;
    const uint32_t padded = xw_pad(Wn) + 1;
    unsigned char* p = base;
    s_x = reinterpret_cast<XT*>(p);
    p += (padded * sizeof(XT) + 15u) & ~15u;
    s_ph = reinterpret_cast<double*>(p);
    p += (padded * 8u + 15u) & ~15u;
    s_pl = reinterpret_cast<float*>(p);
    p += (padded * 4u + 15u) & ~15u;
    s_wt = reinterpret_cast<double*>(p);
  }

  // entries per thread per round: ceil(W / T) capped at kPre, rounded up to
  // even (paired loads); T is a power of two
  static constexpr uint32_t kPre = 8;
  __device__ __forceinline__ uint32_t chunk() const {
    const uint32_t lg = (uint32_t)__ffs((int)T) - 1u;
    const uint32_t e = min(kPre, (W + T - 1u) >> lg);
    return (e + 1u) & ~1u;
  }

  // Loads of a thread's chunk [j0, j0 + E) of the window (zeros past W or n),
  // two entries per load when x is aligned for it.
  __device__ __forceinline__ void load_chunk(uint32_t n, uint32_t j0, uint32_t E, XT (&r)[kPre]) const {
    using P2 = typename std::conditional<sizeof(XT) == 8, double2, float2>::type;
    const bool vec = (reinterpret_cast<uintptr_t>(x) & (2 * sizeof(XT) - 1)) == 0;
#pragma unroll
    for (uint32_t q = 0; q < kPre / 2; ++q) {
      r[2 * q] = XT(0);
      r[2 * q + 1] = XT(0);
      const uint32_t j = j0 + 2 * q, c = wlo + j;
      if (2 * q < E && j < W) {  // W is a multiple of 16 and j even: j + 1 < W
        if (vec && c + 1 < n) {
          const P2 v = __ldg(reinterpret_cast<const P2*>(x + c));
          r[2 * q] = v.x;
          r[2 * q + 1] = v.y;
        } else {
          if (c < n) r[2 * q] = __ldg(x + c);
          if (c + 1 < n) r[2 * q + 1] = __ldg(x + c + 1);
        }
      }
    }
  }

  // Register prefetch of the first round's chunk: issued before the CTA's
  // other setup so the global-load latency overlaps it.
  __device__ __forceinline__ void prefetch(uint32_t n, XT (&r)[kPre]) const {
    load_chunk(n, threadIdx.x * chunk(), chunk(), r);
  }

  // Cooperative staging (all threads of the CTA); ends with __syncthreads().
  __device__ __forceinline__ void stage(uint32_t n) {
    XT r[kPre];
    prefetch(n, r);
    stage(n, r);
  }
  __device__ __forceinline__ void stage(uint32_t n, const XT (&r0)[kPre]) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t E = chunk(), per_round = T * E;
    double ch = 0.0, cl = 0.0;  // carry: the window total before this round (double-double)
    XT r[kPre];
#pragma unroll
    for (uint32_t k = 0; k < kPre; ++k) r[k] = r0[k];
    if (tid == 0) s_x[xw_pad(W)] = XT(0);  // zero entry for padding codes and idle lanes
    for (uint32_t rb = 0; rb < W; rb += per_round) {
      const uint32_t j0 = rb + tid * E;
      if (rb) load_chunk(n, j0, E, r);
      // chunk total (double-double)
      double h = 0.0, l = 0.0;
#pragma unroll
      for (uint32_t k = 0; k < kPre; ++k) {
        if (k < E) {
          double s, e;
          two_sum(h, (double)r[k], s, e);
          h = s;
          l += e;
        }
      }
      // inclusive warp scan of the chunk totals
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const double uh = __shfl_up_sync(0xffffffffu, h, o), ul = __shfl_up_sync(0xffffffffu, l, o);
        if (lane >= o) {
          double s, e;
          two_sum(h, uh, s, e);
          h = s;
          l += ul + e;
        }
      }
      if (lane == 31) {
        s_wt[2 * warp] = h;
        s_wt[2 * warp + 1] = l;
      }
      double ph = __shfl_up_sync(0xffffffffu, h, 1), pl = __shfl_up_sync(0xffffffffu, l, 1);
      if (lane == 0) ph = pl = 0.0;
      __syncthreads();
      // + the totals of the warps before this one, + the carry
      {
        double s, e;
        two_sum(ph, ch, s, e);
        ph = s;
        pl += cl + e;
        for (uint32_t w = 0; w < warp; ++w) {
          two_sum(ph, s_wt[2 * w], s, e);
          ph = s;
          pl += s_wt[2 * w + 1] + e;
        }
      }
      // x and F from registers
#pragma unroll
      for (uint32_t k = 0; k < kPre; ++k) {
        const uint32_t j = j0 + k;
        if (k < E && j < W) {
          const uint32_t p = xw_pad(j);
          s_x[p] = r[k];
          const double hi = ph + pl;
          s_ph[p] = hi;
          s_pl[p] = (float)(pl - (hi - ph));
          double s, e;
          two_sum(ph, (double)r[k], s, e);
          ph = s;
          pl += e;
        }
      }
      // the last thread's running sum is the window total through this round:
      // F[W] after the last round, else the next round's carry
      const bool last = rb + per_round >= W;
      if (tid == T - 1u) {
        if (last) {
          const double hi = ph + pl;
          s_ph[xw_pad(W)] = hi;
          s_pl[xw_pad(W)] = (float)(pl - (hi - ph));
        } else {
          s_wt[2 * 32] = ph;
          s_wt[2 * 32 + 1] = pl;
        }
      }
      __syncthreads();
      if (!last) {
        ch = s_wt[2 * 32];
        cl = s_wt[2 * 32 + 1];
      }
    }
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
