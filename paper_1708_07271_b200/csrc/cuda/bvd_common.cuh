// Shared device pieces of the BV-D product kernels: block staging (TMA bulk
// copy of the coded block), row setup (row bit offsets + warp rounds), code
// extraction, compensated accumulation and the reference-chain level phases.
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
  uint32_t pad;
};

__host__ __device__ inline uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }

// Row-setup scratch carved after the x-window.
struct RowSmem {
  uint32_t off_rowoff, off_perm, off_permi, off_ref, off_dep, off_misc, total;
};
__host__ __device__ inline RowSmem row_smem_layout(uint32_t base, uint32_t B) {
  RowSmem s;
  uint32_t o = base;
  s.off_rowoff = o;
  o = align16(o + B * 4);
  s.off_perm = o;
  o = align16(o + B * 2);
  s.off_permi = o;
  o = align16(o + B * 2);
  s.off_ref = o;
  o = align16(o + B);
  s.off_dep = o;
  o = align16(o + B);
  s.off_misc = o;  // mbarrier (8) + 8 ints + 2 x 64-bin histograms + scratch (64 x 4)
  o = align16(o + 16 + 32 + 128 * 4 + 64 * 4);
  s.total = o;
  return s;
}

struct RowCtx {
  const uint32_t* base;  // block stream (headers at word 0); shared or global
  uint32_t* rowoff;      // bit offset of each row body
  uint16_t* perm;        // rows sorted by point-code count (point rounds)
  uint16_t* permi;       // rows with intervals, sorted by interval count (interval rounds)
  uint8_t* ref;          // reference distance per row
  uint8_t* dep;          // chain depth per row
  int* misc;             // [0] nesc, [1] dmax, [2] rows with intervals, [3] round counter (points),
                         // [4] round counter (intervals)
  int* hist;             // 64 bins (point counts) + 64 bins (interval counts)
  int* wscratch;         // 64 ints (per-warp partials; depth-level starts)
  uint64_t* bar;
  uint32_t nr, B;
};

__device__ __forceinline__ RowCtx carve_rows(unsigned char* smem, const RowSmem& L, uint32_t B, uint32_t nr) {
  RowCtx c;
  c.rowoff = reinterpret_cast<uint32_t*>(smem + L.off_rowoff);
  c.perm = reinterpret_cast<uint16_t*>(smem + L.off_perm);
  c.permi = reinterpret_cast<uint16_t*>(smem + L.off_permi);
  c.ref = reinterpret_cast<uint8_t*>(smem + L.off_ref);
  c.dep = reinterpret_cast<uint8_t*>(smem + L.off_dep);
  c.bar = reinterpret_cast<uint64_t*>(smem + L.off_misc);
  c.misc = reinterpret_cast<int*>(smem + L.off_misc + 16);
  c.hist = reinterpret_cast<int*>(smem + L.off_misc + 48);
  c.wscratch = reinterpret_cast<int*>(smem + L.off_misc + 48 + 512);
  c.B = B;
  c.nr = nr;
  return c;
}

// Issue the TMA bulk copy of the block's coded stream (thread 0).  Blocks
// larger than the staging cap decode straight from global memory.
__device__ __forceinline__ const uint32_t* stage_stream_begin(const BvdDev& g, const BvdBlockInfo& bi, uint32_t* s_stream,
                                                              uint64_t* s_bar) {
  const bool staged = bi.nwords <= g.stream_cap_words;
  if (threadIdx.x == 0) {
    mbar_init(s_bar, 1);
    const uint32_t sbytes = staged ? bi.nwords * 4u : 0u;
    mbar_arrive_expect_tx(s_bar, sbytes);
    if (sbytes) bulk_g2s(s_stream, g.words + bi.word_offset, sbytes, s_bar);
  }
  if (threadIdx.x < 8) s_stream[(staged ? bi.nwords : 0u) + threadIdx.x] = 0u;
  return staged ? s_stream : g.words + bi.word_offset;
}

__device__ __forceinline__ uint32_t extract_bits(const uint32_t* s, uint32_t off, uint32_t w) {
  const uint32_t wi = off >> 5, sh = off & 31u;
  const uint64_t win = (((uint64_t)s[wi] << 32) | s[wi + 1]) << sh;
  return w ? (uint32_t)(win >> (64u - w)) : 0u;
}

__device__ __forceinline__ int32_t unfold32(uint32_t u) {
  return (int32_t)(u >> 1) ^ -(int32_t)(u & 1u);
}

// Row counts (escaped rows look their counts up in the escape table that
// follows the headers: entries (row, #minus, #residual, #interval)).
struct RowCounts {
  uint32_t nm, ns, ni;
};
__device__ __forceinline__ RowCounts row_counts(const uint32_t* base, uint32_t B, uint32_t h, uint32_t k, int nesc) {
  RowCounts c{hdr_nm(h), hdr_ns(h), hdr_ni(h)};
  if (hdr_escaped(h)) {
    const uint32_t* esc = base + B;
    int lo = 0, hi = nesc - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (esc[4 * mid] < k) lo = mid + 1;
      else hi = mid;
    }
    c.nm = esc[4 * lo + 1];
    c.ns = esc[4 * lo + 2];
    c.ni = esc[4 * lo + 3];
  }
  return c;
}

// Row setup, all threads: row bit offsets (exclusive scan of body lengths),
// reference distances, and two warp-round permutations (counting sorts):
// all rows by point-code count, and the rows that have intervals by interval
// count.  Ends with __syncthreads().
__device__ __forceinline__ void row_setup(RowCtx& c) {
  const uint32_t T = blockDim.x, tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, nwarps = T >> 5;
  const uint32_t B = c.B, nr = c.nr;
  const uint32_t per = (B + T - 1) >> (31 - __clz(T));  // contiguous rows per thread (T is a power of 2)
  const uint32_t k0 = tid * per;
  int* hp = c.hist;       // point-count bins
  int* hi = c.hist + 64;  // interval-count bins
  // 1. escape count (rows escape all three counts together)
  int esc_here = 0;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t k = k0 + j;
    if (k < nr && hdr_escaped(c.base[k])) ++esc_here;
  }
  for (uint32_t k = tid; k < 128; k += T) c.hist[k] = 0;
  if (tid < 8) c.misc[tid] = 0;
  const int wsum = __reduce_add_sync(0xffffffffu, esc_here);
  if (lane == 0) c.wscratch[warp] = wsum;
  __syncthreads();
  int nesc = 0;
  for (uint32_t w = 0; w < nwarps; ++w) nesc += c.wscratch[w];
  const uint32_t body0 = (B + 4u * (uint32_t)nesc) * 32u;  // bodies follow headers + escape table
  // 2. body lengths (local scan), ref distances, sort keys
  uint32_t loc = 0;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t k = k0 + j;
    if (k < nr) {
      const uint32_t h = c.base[k];
      const RowCounts rc = row_counts(c.base, B, h, k, nesc);
      c.rowoff[k] = loc;  // local prefix for now
      loc += (rc.nm + rc.ns + rc.ni) * hdr_wp(h) + rc.ni * hdr_wl(h);
      c.ref[k] = (uint8_t)hdr_r(h);
      atomicAdd(&hp[min(rc.nm + rc.ns, 63u)], 1);
      if (rc.ni) atomicAdd(&hi[min(rc.ni, 63u)], 1);
    }
  }
  // 3. block exclusive scan of the per-thread totals
  uint32_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if ((int)lane >= o) inc += u;
  }
  __syncthreads();  // wscratch reuse; histograms complete
  if (lane == 31) c.wscratch[warp] = (int)inc;
  // 4. histogram prefixes (descending keys: longest rows first); warp 0 does
  //    the point bins, warp 1 (or warp 0 again) the interval bins
  for (uint32_t which = warp; which < 2; which += nwarps) {
    int* hb = c.hist + 64 * which;
    const int v0 = hb[63 - 2 * lane], v1 = hb[62 - 2 * lane];
    const int sm = v0 + v1;
    int incs = sm;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incs, o);
      if ((int)lane >= o) incs += u;
    }
    const int ex = incs - sm;
    hb[63 - 2 * lane] = ex;
    hb[62 - 2 * lane] = ex + v0;
    if (which == 1 && lane == 31) c.misc[2] = incs;  // rows with intervals
  }
  __syncthreads();
  uint32_t wbase = 0;
  for (uint32_t w = 0; w < warp; ++w) wbase += (uint32_t)c.wscratch[w];
  const uint32_t tbase = body0 + wbase + inc - loc;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t k = k0 + j;
    if (k < nr) {
      c.rowoff[k] += tbase;
      const uint32_t h = c.base[k];
      const RowCounts rc = row_counts(c.base, B, h, k, nesc);
      c.perm[atomicAdd(&hp[min(rc.nm + rc.ns, 63u)], 1)] = (uint16_t)k;
      if (rc.ni) c.permi[atomicAdd(&hi[min(rc.ni, 63u)], 1)] = (uint16_t)k;
    }
  }
  if (tid == 0) c.misc[0] = nesc;
  __syncthreads();
}

// Neumaier-compensated accumulation (error ~ eps*|sum| + n eps^2 sum|t|):
// keeps y_i accurate to ~1 ulp even when the differential terms cancel.
__device__ __forceinline__ void nadd(double& s, double& c, double t) {
  const double u = s + t;
  const bool big = fabs(s) >= fabs(t);
  const double a = big ? s : t, b = big ? t : s;
  c += (a - u) + b;
  s = u;
}

__device__ __forceinline__ void dd_add(double& hi, double& lo, double bhi, double blo) {
  const double s = hi + bhi;
  const double bb = s - hi;
  const double e = (hi - (s - bb)) + (bhi - bb) + lo + blo;
  hi = s + e;
  lo = e - (hi - s);
}

// Reference-chain resolution -- the level scheduler: rows are counting-
// sorted by chain depth (depth = number of references to the chain root) and
// each level is one barrier-separated data-parallel step,
//     y_i = delta_i + y_{i-r}   (double-double, the reference's order,
//                                ref_matvec.hpp:23-25),
// so every thread does useful work at every level.  Writes y (YT) to global
// memory with coalesced stores.  Reuses perm[] and the histogram.
template <typename YT>
__device__ __forceinline__ void chain_and_store(double* s_yhi, float* s_ylo, RowCtx& c, YT* __restrict__ yb) {
  const uint32_t T = blockDim.x, tid = threadIdx.x, lane = tid & 31u;
  int* hd = c.hist;  // 64 depth bins (deeper chains share bin 63 and are walked in order)
  for (uint32_t k = tid; k < 64; k += T) hd[k] = 0;
  __syncthreads();
  int dmax = 0;
  for (uint32_t k = tid; k < c.nr; k += T) {
    uint32_t d = 0, j = k;
    while (c.ref[j]) {
      j -= c.ref[j];
      ++d;
    }
    c.dep[k] = (uint8_t)min(d, 255u);
    dmax = max(dmax, (int)d);
    atomicAdd(&hd[min(d, 63u)], 1);
  }
  dmax = __reduce_max_sync(0xffffffffu, dmax);
  if (lane == 0 && dmax) atomicMax(&c.misc[1], dmax);
  __syncthreads();
  dmax = c.misc[1];
  if (dmax > 0) {
    if (tid < 32) {  // exclusive scan of the 64 depth bins -> level starts
      const int v0 = hd[2 * lane], v1 = hd[2 * lane + 1];
      const int sm = v0 + v1;
      int inc = sm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)lane >= o) inc += u;
      }
      hd[2 * lane] = inc - sm;
      hd[2 * lane + 1] = inc - sm + v0;
      c.wscratch[2 * lane] = inc - sm;
      c.wscratch[2 * lane + 1] = inc - sm + v0;
    }
    __syncthreads();
    for (uint32_t k = tid; k < c.nr; k += T) c.perm[atomicAdd(&hd[min((uint32_t)c.dep[k], 63u)], 1)] = (uint16_t)k;
    __syncthreads();
    // levels 1..min(dmax, 62): one barrier each
    const int dl = min(dmax, 62);
    for (int d = 1; d <= dl; ++d) {
      const int a = c.wscratch[d], e = c.wscratch[d + 1];
      for (int s = a + (int)tid; s < e; s += (int)T) {
        const uint32_t k = c.perm[s], j = k - c.ref[k];
        double hi = s_yhi[k], lo = s_ylo[k];
        dd_add(hi, lo, s_yhi[j], s_ylo[j]);
        s_yhi[k] = hi;
        s_ylo[k] = (float)lo;
      }
      __syncthreads();
    }
    if (dmax >= 63) {  // chains deeper than 62: bin 63 walked in row order by one thread
      if (tid == 0) {
        const int a = c.wscratch[63];
        for (uint32_t k = 0; k < c.nr; ++k)
          if (c.dep[k] >= 63) {
            const uint32_t j = k - c.ref[k];
            double hi = s_yhi[k], lo = s_ylo[k];
            dd_add(hi, lo, s_yhi[j], s_ylo[j]);
            s_yhi[k] = hi;
            s_ylo[k] = (float)lo;
          }
        (void)a;
      }
      __syncthreads();
    }
  }
  for (uint32_t k = tid; k < c.nr; k += T) yb[k] = (YT)(s_yhi[k] + (double)s_ylo[k]);
}

}  // namespace cmvg
