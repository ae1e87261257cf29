// Shared device pieces of the product kernels: the block table view, code
// extraction from row-major bit-packed bodies (heavy rows), compensated
// accumulation, the PageRank epilogue and the reference-chain resolution.
// Layouts: host/layout.hpp.
#pragma once
#include <cstdint>

#include "../host/layout.hpp"
#include "ptx.cuh"
#include "xwindow.cuh"

namespace cmvg {

struct BvdDev {
  const uint32_t* words;
  const BvdBlockInfo* blocks;
  BvdDims d;
  uint32_t block_begin;       // first block of this shard
  uint32_t row_begin;         // first row of this shard
  uint32_t stream_cap_words;  // blocks with more words decode from global memory
  uint32_t nlaunch;           // blocks of this launch (`blocks` is offset to its first)
  uint32_t ahead;             // L2 prefetch distance in blocks (resident CTAs of the launch; 0 = none)
  uint32_t pad_[3];
  double2* hpart;             // heavy-row work-item partial sums (BV-S), indexed by the global item number
};

__host__ __device__ inline uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }

// ---- coded-stream source: the block's words in global memory (read through L1/L2)
template <bool STAGED>
struct Src;
template <>
struct Src<false> {
  const uint32_t* __restrict__ p;
  __device__ __forceinline__ uint32_t w(uint32_t i) const { return __ldg(p + i); }
};

template <class S>
__device__ __forceinline__ uint32_t extract_bits(const S& s, uint32_t off, uint32_t w) {
  const uint32_t wi = off >> 5, sh = off & 31u;
  const uint64_t win = (((uint64_t)s.w(wi) << 32) | s.w(wi + 1)) << sh;
  return w ? (uint32_t)(win >> (64u - w)) : 0u;
}

// ---- a block row's record in shared memory: its delta (double-double, lo
// rounded to fp32) and reference distance, 16 bytes, so the slice epilogue
// writes it with one 16-byte store and the chain walk reads an ancestor with
// one 16-byte load
struct __align__(16) RowRec {
  double hi;
  float lo;
  uint32_t ref;
};
__device__ __forceinline__ void put_row(RowRec* rows, uint32_t k, double hi, double lo, uint32_t r) {
  double2 v;
  v.x = hi;
  v.y = __hiloint2double((int)r, __float_as_int((float)lo));  // {lo, ref} as the record's second 8 bytes
  *reinterpret_cast<double2*>(rows + k) = v;
}

// ---- reference-chain context of a block (chain_and_store) --------------------
struct ChainCtx {
  RowRec* rows;    // per row of the block: delta and reference distance
  uint16_t* ptr;   // scratch: chain pointers (unbounded chains only)
  int* wscratch;   // 64 ints: epilogue reductions
  uint32_t nr;     // rows in the block
};

// Compensated accumulation: TwoSum, error term into `c` (error ~ eps|sum| +
// n eps^2 sum|t|), so y_i stays accurate when the differential terms cancel.
__device__ __forceinline__ void tsum(double& s, double& c, double t) {
  const double u = s + t;
  const double bb = u - s;
  c += (s - (u - bb)) + (t - bb);
  s = u;
}

__device__ __forceinline__ void dd_add(double& hi, double& lo, double bhi, double blo) {
  const double s = hi + bhi;
  const double bb = s - hi;
  const double e = (hi - (s - bb)) + (bhi - bb) + lo + blo;
  hi = s + e;
  lo = e - (hi - s);
}

// Output stage of the gather: plain y, or the fused PageRank update
// (pagerank.hpp:83-102, Eq. 1):
//   p'_i = alpha/n + (1 - alpha) (y_i + D/n)   (D = dangling mass, kUniform;
//                                                0 for kDrop)
//   q'_i = p'_i / d_i  (0 for dangling i)
// plus per-block partials {sum_{d_i = 0} p'_i, sum |p'_i - p_i|}.
// An epilogue's per-row inputs are loaded for a thread's kEpiPre rows at
// once (prefetch), before their chain walks, so the global-load latency
// overlaps the walks instead of stalling each row's store.
constexpr uint32_t kEpiPre = 4;

struct PlainEpi {
  __device__ __forceinline__ void prefetch(uint32_t, uint32_t, uint32_t) {}
  template <typename YT>
  __device__ __forceinline__ void store(YT* yb, uint32_t k, double y, uint32_t) const {
    yb[k] = (YT)y;
  }
  __device__ __forceinline__ void finish(int*) const {}
};

struct PageRankEpi {
  const uint32_t* deg;     // out-degrees of A for this block's rows (shard-relative, offset applied)
  const double* p_prev;    // may be null
  double* q_next;          // shard-relative, offset applied
  double* partial;         // [nblocks][2]
  double base, scale, dn;  // alpha/n, 1 - alpha, D/n (or 0)
  double alpha_p0;         // alpha (multiplies p0 when a restart distribution is given)
  uint32_t bl;
  double dang, l1;         // per-thread partials
  // fused halo push (multi-GPU): q'_k also goes to every peer whose bit is set
  // in push_mask[k], stored at its global column in that peer's q buffer
  // (NVLink peer memory) -- the exchange rides on the epilogue's stores
  const double* p0;            // restart distribution of this block's rows (offset applied); null = uniform
  const uint8_t* push_mask;    // shard-relative, offset applied; null = no push
  double* const* push_dst;     // device array: peer q buffers, indexed by global column
  uint32_t grow0;              // global row of this block's row 0
  uint32_t dpre[kEpiPre];      // prefetched d_k of the thread's next rows (p0 / p_prev are optional: loaded in place)
  __device__ __forceinline__ void prefetch(uint32_t k0, uint32_t T, uint32_t nr) {
#pragma unroll
    for (uint32_t q = 0; q < kEpiPre; ++q) {
      const uint32_t k = k0 + q * T;
      dpre[q] = k < nr ? __ldg(deg + k) : 0u;
    }
  }
  template <typename YT>
  __device__ __forceinline__ void store(YT* pb, uint32_t k, double y, uint32_t q) {
    const double pn = (p0 ? alpha_p0 * p0[k] : base) + scale * (y + dn);
    pb[k] = (YT)pn;
    const uint32_t d = dpre[q];
    const double qn = d ? pn / (double)d : 0.0;
    q_next[k] = qn;
    if (push_mask) {
      uint32_t m = push_mask[k];
      while (m) {
        const uint32_t p = (uint32_t)__ffs(m) - 1u;
        m &= m - 1u;
        push_dst[p][grow0 + k] = qn;
      }
    }
    if (!d) dang += pn;
    if (p_prev) l1 += fabs(pn - p_prev[k]);
  }
  __device__ __forceinline__ void finish(int* scratch) {
    if (push_mask) __threadfence_system();  // peer stores performed before the kernel's completion is observed
    // deterministic block reduction: warp sums, then warp 0 in warp order
    double a = dang, b = l1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
    }
    double* ws = reinterpret_cast<double*>(scratch);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) {
      ws[2 * warp] = a;
      ws[2 * warp + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sa = 0.0, sb = 0.0;
      for (uint32_t w = 0; w < nw; ++w) {
        sa += ws[2 * w];
        sb += ws[2 * w + 1];
      }
      partial[2 * bl] = sa;
      partial[2 * bl + 1] = sb;
    }
  }
};

// Reference-chain resolution -- the level scheduler.  Every row holds
// (value, pointer) = (delta_i, i - r_i); each level of pointer jumping is one
// barrier-separated data-parallel step
//     value_i += value_{ptr_i};  ptr_i = ptr_{ptr_i}
// in double-double, so after ceil(log2(depth + 1)) levels value_i = y_i =
// delta_i + y_{i - r_i} (ref_matvec.hpp:23-25; the pairing differs from the
// reference's left-to-right order only below double-double resolution).
// Bounded chains (R = 3) take two levels; unbounded ones log2(depth).
// Writes y (YT) with coalesced stores.  Uses c.ptr as the pointer array.
template <typename YT, class EPI = PlainEpi>
__device__ __forceinline__ void chain_and_store(const ChainCtx& c, YT* __restrict__ yb, EPI epi = EPI(),
                                                uint32_t max_depth = 0xffffffffu, uint32_t T = blockDim.x) {
  const uint32_t tid = threadIdx.x;
  RowRec* rows = c.rows;
  if (max_depth <= 3) {
    // Bounded chains (R <= 3): each row walks its <= 3 ancestors,
    // y_i = d_i + d_p1 + d_p2 + d_p3 accumulated with TwoSum (error terms
    // collected with the low parts), no barriers; one 16-byte load per row.
    for (uint32_t kb = tid; kb < c.nr; kb += kEpiPre * T) {
      epi.prefetch(kb, T, c.nr);
#pragma unroll
      for (uint32_t q = 0; q < kEpiPre; ++q) {
        const uint32_t k = kb + q * T;
        if (k >= c.nr) break;
        const RowRec rk = rows[k];
        double s = rk.hi, e = (double)rk.lo;
        uint32_t p = k, r = rk.ref;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          if (r) {
            p -= r;
            const RowRec rp = rows[p];
            tsum(s, e, rp.hi);
            e += (double)rp.lo;
            r = rp.ref;
          }
        }
        epi.store(yb, k, s + e, q);
      }
    }
    epi.finish(c.wscratch);
    return;
  }
  constexpr uint32_t kMaxPer = 4;  // rows per thread per level (block_rows / threads <= 4)
  constexpr uint16_t kNone = 0xffffu;
  uint16_t* ptr = c.ptr;
  int any = 0;
  for (uint32_t k = tid; k < c.nr; k += T) {
    const uint32_t r = rows[k].ref;
    ptr[k] = r ? (uint16_t)(k - r) : kNone;
    any |= (r != 0);
  }
  any = __syncthreads_or(any);
  while (any) {
    double nh[kMaxPer], nl[kMaxPer];
    uint16_t np_[kMaxPer];
    int more = 0;
#pragma unroll
    for (uint32_t q = 0; q < kMaxPer; ++q) {
      const uint32_t k = tid + q * T;
      if (k < c.nr) {
        const uint32_t p = ptr[k];
        double h = rows[k].hi, l = rows[k].lo;
        uint16_t pn = kNone;
        if (p != kNone) {
          dd_add(h, l, rows[p].hi, rows[p].lo);
          pn = ptr[p];
        }
        nh[q] = h;
        nl[q] = l;
        np_[q] = pn;
        more |= (pn != kNone);
      }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t q = 0; q < kMaxPer; ++q) {
      const uint32_t k = tid + q * T;
      if (k < c.nr) {
        rows[k].hi = nh[q];
        rows[k].lo = (float)nl[q];
        ptr[k] = np_[q];
      }
    }
    any = __syncthreads_or(more);
  }
  for (uint32_t kb = tid; kb < c.nr; kb += kEpiPre * T) {
    epi.prefetch(kb, T, c.nr);
#pragma unroll
    for (uint32_t q = 0; q < kEpiPre; ++q) {
      const uint32_t k = kb + q * T;
      if (k < c.nr) epi.store(yb, k, rows[k].hi + (double)rows[k].lo, q);
    }
  }
  epi.finish(c.wscratch);
}

}  // namespace cmvg
