// bv_decode_csr: canonical BV stream -> CSR on the device, bit-exact with the
// source adjacency (the GPU counterpart of `reconstruct_graph`,
// reference include/cmv/ref_matrix.hpp:75-76, with BV copy blocks resolved
// positionally against the decoded reference list).
//
// Segments are chain-closed, so they decode independently (parallel decoder
// below; bv_seg_decode is the serial thread-per-segment form, kept as the
// cross-check of the tests).
#pragma once
#include <cstdint>

#include "bitreader.cuh"

namespace cmvg {

struct BvDev {
  const uint32_t* words;
  const uint64_t* seg_bits;  // nseg + 1
  uint32_t n;
  uint32_t seg_rows;
  uint32_t nseg;
  uint32_t window;
  uint32_t min_interval;
  uint32_t zeta_k;
};

// Skip the copy-block list; returns the number of copied entries.
__device__ __forceinline__ uint64_t bv_skip_blocks(PosBits& br, uint64_t dr) {
  uint64_t b = br.gamma();
  uint64_t pos = 0, copied = 0;
  bool cp = true;
  for (uint64_t k = 0; k < b; ++k) {
    uint64_t len = k == 0 ? br.gamma() : br.gamma() + 1;
    if (cp) copied += len;
    pos += len;
    cp = !cp;
  }
  if (cp && dr > pos) copied += dr - pos;
  return copied;
}

struct CopyCursor {
  const uint32_t* R;
  uint64_t dr, pos, run_left, nb_left;
  PosBits br;
  bool cp, has;
  uint32_t val;
  __device__ void load_run() {  // next block length
    if (nb_left) {
      run_left = br.gamma() + 1;
      --nb_left;
    } else {
      run_left = dr - pos;
    }
  }
  __device__ void advance() {
    for (;;) {
      if (run_left == 0) {
        if (pos >= dr) { has = false; return; }
        cp = !cp;
        load_run();
        continue;
      }
      if (cp) {
        val = R[pos++];
        --run_left;
        has = true;
        return;
      }
      pos += run_left;
      run_left = 0;
    }
  }
};

// One row, serially (one thread): row i starts at bit position br.pos; its
// columns go to cols[off, off + d).  Returns false on a corrupt stream.
__device__ __forceinline__ bool bv_decode_row_serial(const BvDev& s, uint32_t i, PosBits& br, uint64_t off,
                                                     const uint64_t* __restrict__ row_offsets,
                                                     uint32_t* __restrict__ cols, int* __restrict__ err) {
  uint64_t d = br.gamma();
  if (d == 0) return true;
  uint32_t r = s.window ? br.unary() : 0u;
  CopyCursor cc;
  cc.has = false;
  uint64_t copied = 0;
  if (r) {
    uint32_t j = i - r;
    uint64_t rb = row_offsets[j], re = row_offsets[j + 1];
    cc.R = cols + rb;
    cc.dr = re - rb;
    PosBits probe = br;
    copied = bv_skip_blocks(probe, cc.dr);
    // the cursor re-reads the block list lazily
    cc.br = br;
    uint64_t b = cc.br.gamma();
    cc.pos = 0;
    cc.cp = true;
    if (b) {
      cc.run_left = cc.br.gamma();
      cc.nb_left = b - 1;
    } else {
      cc.nb_left = 0;
      cc.run_left = cc.dr;
    }
    cc.advance();
    br = probe;
  }
  uint64_t extra = d - copied;
  // interval cursor and residual cursor
  uint64_t ni = 0, in_int = 0;
  PosBits ib = br;
  if (extra) {
    ni = ib.gamma();
    br = ib;
    for (uint64_t k = 0; k < ni; ++k) {
      br.gamma();
      in_int += br.gamma() + s.min_interval;
    }
  }
  uint64_t nres = extra - in_int;
  uint64_t int_left = 0, int_len = 0, int_k = 0, int_prev_end = 0, int_t = 0;
  bool ihas = false;
  auto next_interval = [&]() {
    if (int_k >= ni) { ihas = false; return; }
    int64_t left = int_k == 0 ? (int64_t)i + unfold_i32((uint32_t)ib.gamma()) : (int64_t)(int_prev_end + ib.gamma() + 1);
    int_left = (uint64_t)left;
    int_len = ib.gamma() + s.min_interval;
    int_prev_end = int_left + int_len;
    int_t = 0;
    ++int_k;
    ihas = true;
  };
  next_interval();
  uint64_t res_k = 0;
  int64_t res_val = 0;
  bool rhas = false;
  auto next_res = [&]() {
    if (res_k >= nres) { rhas = false; return; }
    res_val = res_k == 0 ? (int64_t)i + unfold_i32((uint32_t)br.zeta(s.zeta_k)) : res_val + (int64_t)br.zeta(s.zeta_k) + 1;
    ++res_k;
    rhas = true;
  };
  next_res();
  uint64_t written = 0;
  uint32_t prev = 0;
  while (cc.has || ihas || rhas) {
    uint64_t vc = cc.has ? cc.val : ~0ull;
    uint64_t vi = ihas ? int_left + int_t : ~0ull;
    uint64_t vr = rhas ? (uint64_t)res_val : ~0ull;
    uint64_t v;
    if (vc <= vi && vc <= vr) {
      v = vc;
      cc.advance();
    } else if (vi <= vr) {
      v = vi;
      if (++int_t >= int_len) next_interval();
    } else {
      v = vr;
      next_res();
    }
    if (v >= s.n || (written && v <= prev) || written >= d) { atomicExch(err, 5); return false; }
    cols[off + written] = (uint32_t)v;
    prev = (uint32_t)v;
    ++written;
  }
  if (written != d) { atomicExch(err, 6); return false; }
  return true;
}

// Serial reference decoder: one thread per segment (kept for testing the
// warp-cooperative decoder against).
__global__ void bv_seg_decode(BvDev s, const uint64_t* __restrict__ seg_base, uint64_t* __restrict__ row_offsets,
                              uint32_t* __restrict__ cols, int* __restrict__ err) {
  uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x;
  if (sg >= s.nseg || *(volatile int*)err) return;
  uint32_t r0 = sg * s.seg_rows;
  uint32_t r1 = min(s.n, r0 + s.seg_rows);
  PosBits br{s.words, s.seg_bits[sg]};
  uint64_t off = seg_base[sg];
  for (uint32_t i = r0; i < r1; ++i) {
    row_offsets[i] = off;
    PosBits pk = br;
    const uint64_t d = pk.gamma();
    if (!bv_decode_row_serial(s, i, br, off, row_offsets, cols, err)) return;
    off += d;
  }
  if (br.pos != s.seg_bits[sg + 1]) atomicExch(err, 7);
  if (sg == s.nseg - 1) row_offsets[s.n] = off;
}

// ---------------------------------------------------------------------------
// Parallel decoder (three launches, no host round trip):
//   1. bv_index_rows, one thread per segment: parse the segment (its codes are
//      instantaneous, so this is the one serial step), recording each row's
//      bit position and out-degree, and the segment's edge count;
//   2. bv_scan_segments, one CTA: exclusive scan of the segment edge counts
//      (checked against m);
//   3. bv_decode_tiles, one CTA per tile of 1024 rows (whole segments, so
//      reference chains stay inside): a CTA scan of the degrees gives the
//      rows' offsets; then in rounds, every row whose reference is already
//      decoded is decoded by one thread from its own bit position -- copy
//      blocks over the reference's decoded list, intervals and zeta residuals
//      merged in order -- into a shared-memory staging buffer (references are
//      read from it), which is written out coalesced at the end.  Rounds =
//      the longest reference chain + 1 (<= R + 1).  Tiles with more edges than
//      the buffer decode straight into the output columns.

// One row's decode in two warp-friendly phases, so that the 32 lanes of a
// warp, each on its own row, step together in warp-uniform loops:
//   phase 1: the extra list (BV intervals expanded, merged with the zeta
//            residuals) into the tail of the row's output, out[copied, d);
//   phase 2: merge in place with the copied entries (copy blocks over the
//            decoded reference list R of dr entries): a write never passes
//            the next unread extra, since it lags it by the copies left.
struct RowDec {
  DevBits br, bb, ib;  // residual, copy-block and interval cursors
  const uint32_t* R;
  uint32_t* out;
  uint32_t i, d, r, dr, copied, extra, w, e, nres, rk, ni, ik, ileft, ilen, it, iend, cpos, run, bleft, cval, lmin;
  int64_t rval, prev;
  bool ccp, chas, ihas, rhas;

  // parse the row's header from bit position `bit`; false (err set) on a corrupt stream
  __device__ __forceinline__ bool init(const BvDev& s, uint32_t row, uint64_t bit, uint32_t dexp, uint32_t* o,
                                       const uint32_t* Rl, uint32_t drl, int* __restrict__ err) {
    i = row;
    out = o;
    R = Rl;
    dr = drl;
    lmin = s.min_interval;
    w = 0;
    e = 0;
    copied = extra = 0;
    r = 0;
    prev = -1;
    chas = ihas = rhas = false;
    br.init_bit(s.words, bit);
    d = br.gamma();
    if (d != dexp) { atomicExch(err, 10); return false; }
    if (d == 0) return true;
    r = s.window ? br.unary() : 0u;
    uint32_t nb = 0;
    bb = br;
    if (r) {
      nb = br.gamma();
      bb = br;  // at the first block length
      uint32_t pos = 0;
      bool cp = true;
      for (uint32_t k = 0; k < nb; ++k) {
        const uint32_t len = k == 0 ? br.gamma() : br.gamma() + 1u;
        if (cp) copied += len;
        pos += len;
        cp = !cp;
      }
      if (pos > dr) { atomicExch(err, 12); return false; }
      if (cp) copied += dr - pos;
    }
    if (copied > d) { atomicExch(err, 2); return false; }
    extra = d - copied;
    uint32_t in_int = 0;
    ni = 0;
    ib = br;
    if (extra) {
      ni = br.gamma();
      ib = br;
      for (uint32_t k = 0; k < ni; ++k) {
        br.gamma();
        in_int += br.gamma() + lmin;
      }
    }
    if (in_int > extra) { atomicExch(err, 3); return false; }
    nres = extra - in_int;
    cpos = 0;
    run = 0;
    bleft = 0;
    ccp = true;
    if (r) {
      if (nb) {
        run = bb.gamma();
        bleft = nb - 1;
      } else {
        run = dr;
      }
    }
    ik = 0;
    iadv();
    rk = 0;
    radv();
    return true;
  }
  __device__ __forceinline__ void cadv() {
    chas = false;
    if (!r) return;
    for (;;) {
      if (run == 0) {
        if (cpos >= dr) return;
        ccp = !ccp;
        if (bleft) {
          run = bb.gamma() + 1u;
          --bleft;
        } else {
          run = dr - cpos;
        }
        continue;
      }
      if (ccp) {
        cval = R[cpos++];
        --run;
        chas = true;
        return;
      }
      cpos += run;
      run = 0;
    }
  }
  __device__ __forceinline__ void iadv() {
    if (ik >= ni) { ihas = false; return; }
    ileft = ik == 0 ? (uint32_t)((int64_t)i + unfold_i32(ib.gamma())) : iend + ib.gamma() + 1u;
    ilen = ib.gamma() + lmin;
    iend = ileft + ilen;
    it = 0;
    ++ik;
    ihas = true;
  }
  __device__ __forceinline__ void radv() {
    if (rk >= nres) { rhas = false; return; }
    rval = rk == 0 ? (int64_t)i + unfold_i32(br.zeta<3>()) : rval + (int64_t)br.zeta<3>() + 1;
    ++rk;
    rhas = true;
  }
  __device__ __forceinline__ bool more1() const { return ihas || rhas; }
  // phase 1: the next extra entry into out[copied + e]; false (err set) on a corrupt stream
  __device__ __forceinline__ bool step1(uint32_t n, int* __restrict__ err) {
    const uint64_t vi = ihas ? (uint64_t)ileft + it : ~0ull;
    const uint64_t vr = rhas ? (rval >= 0 ? (uint64_t)rval : ~0ull - 1) : ~0ull;
    uint64_t v;
    if (vi <= vr) {
      v = vi;
      if (++it >= ilen) iadv();
    } else {
      v = vr;
      radv();
    }
    if (v >= n || (int64_t)v <= prev || e >= extra) {
      atomicExch(err, 5);
      ihas = rhas = false;
      return false;
    }
    out[copied + e++] = (uint32_t)v;
    prev = (int64_t)v;
    return true;
  }
  // between the phases
  __device__ __forceinline__ void start2() {
    e = 0;
    prev = -1;
    cadv();
  }
  __device__ __forceinline__ bool more2() const { return chas || e < extra; }
  // phase 2: the smaller of the next copied and the next extra entry into out[w]
  __device__ __forceinline__ bool step2(uint32_t n, int* __restrict__ err) {
    const uint64_t ve = e < extra ? (uint64_t)out[copied + e] : ~0ull;
    const uint64_t vc = chas ? cval : ~0ull;
    uint64_t v;
    if (vc < ve) {
      v = vc;
      cadv();
    } else {
      v = ve;
      ++e;
    }
    if (v >= n || (int64_t)v <= prev || w >= d) {
      atomicExch(err, 5);
      chas = false;
      e = extra;
      return false;
    }
    out[w++] = (uint32_t)v;
    prev = (int64_t)v;
    return true;
  }
  // after the last step: all d columns written, the codes end at next_bit
  __device__ __forceinline__ void finish(const BvDev& s, uint64_t next_bit, int* __restrict__ err) const {
    if (w != d) atomicExch(err, 6);
    else if (br.bitpos(s.words) != next_bit) atomicExch(err, 11);
  }
};

__global__ void bv_index_rows(BvDev s, uint32_t* __restrict__ deg, uint64_t* __restrict__ rbit,
                              uint64_t* __restrict__ seg_edges, int* __restrict__ err) {
  const uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x;
  if (sg >= s.nseg) return;
  const uint32_t r0 = sg * s.seg_rows, r1 = min(s.n, r0 + s.seg_rows);
  DevBits br;
  br.init_bit(s.words, s.seg_bits[sg]);
  uint64_t tot = 0;
  for (uint32_t i = r0; i < r1; ++i) {
    rbit[i] = br.bitpos(s.words);
    const uint32_t d = br.gamma();
    deg[i] = d;
    tot += d;
    if (d == 0) continue;
    const uint32_t r = s.window ? br.unary() : 0u;
    uint32_t copied = 0;
    if (r) {
      if (r > s.window || i < r0 + r) { atomicExch(err, 1); return; }
      const uint32_t dr = deg[i - r];
      const uint32_t b = br.gamma();
      uint32_t pos = 0;
      bool cp = true;
      for (uint32_t k = 0; k < b; ++k) {
        const uint32_t len = k == 0 ? br.gamma() : br.gamma() + 1u;
        if (cp) copied += len;
        pos += len;
        cp = !cp;
      }
      if (pos > dr) { atomicExch(err, 12); return; }
      if (cp) copied += dr - pos;
    }
    if (copied > d) { atomicExch(err, 2); return; }
    const uint32_t extra = d - copied;
    if (extra) {
      const uint32_t ni = br.gamma();
      uint32_t in_int = 0;
      for (uint32_t k = 0; k < ni; ++k) {
        br.gamma();
        in_int += br.gamma() + s.min_interval;
      }
      if (in_int > extra) { atomicExch(err, 3); return; }
      for (uint32_t k = in_int; k < extra; ++k) br.zeta<3>();
    }
  }
  if (br.bitpos(s.words) != s.seg_bits[sg + 1]) atomicExch(err, 4);
  seg_edges[sg] = tot;
}

// Row-group index of a handle (built once, by one serial pass per segment):
// for every kDecGroup-th row its bit position and the out-degrees of the 7
// rows before it (a reference reaches back at most w <= 7 rows, and its
// degree is needed to parse the copy blocks), so that groups parse in parallel.
constexpr uint32_t kDecGroup = 64;
struct __align__(8) DecSync {
  uint64_t bit;
  uint32_t deg[7];
  uint32_t pad;
};

__global__ void bv_sync_index(BvDev s, uint32_t* __restrict__ degscr, DecSync* __restrict__ sync,
                              int* __restrict__ err) {
  const uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x;
  if (sg >= s.nseg) return;
  const uint32_t r0 = sg * s.seg_rows, r1 = min(s.n, r0 + s.seg_rows);
  DevBits br;
  br.init_bit(s.words, s.seg_bits[sg]);
  for (uint32_t i = r0; i < r1; ++i) {
    if (i % kDecGroup == 0) {
      DecSync q;
      q.bit = br.bitpos(s.words);
#pragma unroll
      for (uint32_t k = 0; k < 7; ++k) q.deg[k] = (i >= r0 + 7 - k) ? degscr[i - 7 + k] : 0u;
      q.pad = 0;
      sync[i / kDecGroup] = q;
    }
    const uint32_t d = br.gamma();
    degscr[i] = d;
    if (d == 0) continue;
    const uint32_t r = s.window ? br.unary() : 0u;
    uint32_t copied = 0;
    if (r) {
      if (r > s.window || i < r0 + r) { atomicExch(err, 1); return; }
      const uint32_t dr = degscr[i - r];
      const uint32_t b = br.gamma();
      uint32_t pos = 0;
      bool cp = true;
      for (uint32_t k = 0; k < b; ++k) {
        const uint32_t len = k == 0 ? br.gamma() : br.gamma() + 1u;
        if (cp) copied += len;
        pos += len;
        cp = !cp;
      }
      if (pos > dr) { atomicExch(err, 12); return; }
      if (cp) copied += dr - pos;
    }
    if (copied > d) { atomicExch(err, 2); return; }
    const uint32_t extra = d - copied;
    if (extra) {
      const uint32_t ni = br.gamma();
      uint32_t in_int = 0;
      for (uint32_t k = 0; k < ni; ++k) {
        br.gamma();
        in_int += br.gamma() + s.min_interval;
      }
      if (in_int > extra) { atomicExch(err, 3); return; }
      for (uint32_t k = in_int; k < extra; ++k) br.zeta<3>();
    }
  }
  if (br.bitpos(s.words) != s.seg_bits[sg + 1]) atomicExch(err, 4);
}

// One thread per group of kDecGroup rows: each row's bit position and degree,
// the group's edge count; the parse must end where the next group starts.
__global__ void bv_index_groups(BvDev s, const DecSync* __restrict__ sync, uint32_t* __restrict__ deg,
                                uint64_t* __restrict__ rbit, uint64_t* __restrict__ gcnt, int* __restrict__ err) {
  const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ng = (s.n + kDecGroup - 1) / kDecGroup;
  if (gi >= ng) return;
  const uint32_t r0 = gi * kDecGroup, r1 = min(s.n, r0 + kDecGroup);
  const DecSync q = sync[gi];
  DevBits br;
  br.init_bit(s.words, q.bit);
  uint32_t dl[kDecGroup];  // this group's degrees (local memory; the references' come from here or q.deg)
  uint64_t tot = 0;
  for (uint32_t i = r0; i < r1; ++i) {
    const uint32_t k = i - r0;
    rbit[i] = br.bitpos(s.words);
    const uint32_t d = br.gamma();
    deg[i] = d;
    dl[k] = d;
    tot += d;
    if (d == 0) continue;
    const uint32_t r = s.window ? br.unary() : 0u;
    uint32_t copied = 0;
    if (r) {
      if (r > s.window || (i % s.seg_rows) < r) { atomicExch(err, 1); return; }
      const uint32_t dr = r <= k ? dl[k - r] : q.deg[7 + k - r];
      const uint32_t b = br.gamma();
      uint32_t pos = 0;
      bool cp = true;
      for (uint32_t t = 0; t < b; ++t) {
        const uint32_t len = t == 0 ? br.gamma() : br.gamma() + 1u;
        if (cp) copied += len;
        pos += len;
        cp = !cp;
      }
      if (pos > dr) { atomicExch(err, 12); return; }
      if (cp) copied += dr - pos;
    }
    if (copied > d) { atomicExch(err, 2); return; }
    const uint32_t extra = d - copied;
    if (extra) {
      const uint32_t ni = br.gamma();
      uint32_t in_int = 0;
      for (uint32_t t = 0; t < ni; ++t) {
        br.gamma();
        in_int += br.gamma() + s.min_interval;
      }
      if (in_int > extra) { atomicExch(err, 3); return; }
      for (uint32_t t = in_int; t < extra; ++t) br.zeta<3>();
    }
  }
  const uint64_t end = gi + 1 < ng ? sync[gi + 1].bit : s.seg_bits[s.nseg];
  if (br.bitpos(s.words) != end) atomicExch(err, 4);
  gcnt[gi] = tot;
}

// exclusive scan, in one CTA of 1024 threads, of per-unit edge counts summed
// G units at a time (G = 1: per segment; G = tile rows / group rows: per tile);
// rounds of 1024 sums, coalesced; the total must be m
__global__ void __launch_bounds__(1024) bv_scan_segments(const uint64_t* __restrict__ cnt, uint64_t nunit, uint32_t G,
                                                         uint64_t m, uint64_t* __restrict__ base,
                                                         int* __restrict__ err) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t carry;
  const uint32_t t = threadIdx.x, lane = t & 31u, w = t >> 5;
  const uint64_t nout = (nunit + G - 1) / G;
  if (t == 0) carry = 0;
  __syncthreads();
  for (uint64_t b0 = 0; b0 < nout; b0 += 1024) {
    const uint64_t o = b0 + t;
    uint64_t sum = 0;
    if (o < nout)
      for (uint64_t u = o * G; u < min(nunit, (o + 1) * G); ++u) sum += cnt[u];
    uint64_t inc = sum;
#pragma unroll
    for (int q = 1; q < 32; q <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, inc, q);
      if (lane >= (uint32_t)q) inc += u;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
      const uint64_t v = ws[lane];
      uint64_t iv = v;
#pragma unroll
      for (int q = 1; q < 32; q <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, iv, q);
        if (lane >= (uint32_t)q) iv += u;
      }
      ws[lane] = iv - v;
    }
    __syncthreads();
    const uint64_t c = carry;
    if (o < nout) base[o] = c + ws[w] + inc - sum;
    __syncthreads();
    if (t == 1023) carry = c + ws[w] + inc;
    __syncthreads();
  }
  if (t == 0 && carry != m) atomicExch(err, 13);  // decoded edge count != m
}

constexpr uint32_t kDecTileRows = 1024, kDecThreads = 256;
// shared memory of bv_decode_tiles: loff[T + 1] u32, lvl[T + 2] u32,
// order[T] u16, dep[T] u16, r[T] u8, then the staging buffer
__host__ __device__ constexpr uint32_t dec_smem_bytes(uint32_t cap_words) {
  return ((kDecTileRows + 1) * 4 + (kDecTileRows + 2) * 4 + kDecTileRows * 5 + 15) / 16 * 16 + cap_words * 4;
}

// One CTA per tile of kDecTileRows rows (whole segments).  Rows are sorted by
// reference depth (counting sort in shared memory); each depth level is one
// barrier-separated phase whose rows the warps take from a shared queue, a
// lane taking the next row as soon as its current one is done.
__global__ void __launch_bounds__(kDecThreads, 4) bv_decode_tiles(BvDev s, const uint32_t* __restrict__ deg,
                                                               const uint64_t* __restrict__ rbit,
                                                               const uint64_t* __restrict__ tile_base, uint32_t cap,
                                                               uint64_t* __restrict__ row_offsets,
                                                               uint32_t* __restrict__ cols, int* __restrict__ err,
                                                               uint8_t* __restrict__ ref_out = nullptr) {
  constexpr uint32_t T = kDecTileRows;
  extern __shared__ __align__(16) unsigned char dsm[];
  uint32_t* loff = reinterpret_cast<uint32_t*>(dsm);  // [T + 1]
  uint32_t* lvl = loff + (T + 1);                     // [T + 2]: level starts (counts first)
  uint16_t* order = reinterpret_cast<uint16_t*>(lvl + (T + 2));
  uint16_t* dep = order + T;
  uint8_t* rr = reinterpret_cast<uint8_t*>(dep + T);
  uint32_t* buf = reinterpret_cast<uint32_t*>(dsm + ((T + 1) * 4 + (T + 2) * 4 + T * 5 + 15) / 16 * 16);
  __shared__ uint32_t wsum[kDecThreads / 32];
  __shared__ uint32_t nlev;
  if (*(volatile int*)err) return;  // the index pass or the scan found the stream corrupt
  const uint32_t t = threadIdx.x, lane = t & 31u, w = t >> 5;
  const uint32_t r0 = blockIdx.x * T, nr = min(T, s.n - r0);
  const uint64_t base = tile_base[blockIdx.x];
  // local row offsets (CTA scan of the degrees) and each row's reference distance
  constexpr uint32_t RPT = T / kDecThreads;
  const uint32_t k0 = RPT * t;
  uint32_t dv[RPT], sum = 0;
#pragma unroll
  for (uint32_t q = 0; q < RPT; ++q) {
    const uint32_t k = k0 + q;
    dv[q] = k < nr ? deg[r0 + k] : 0u;
    sum += dv[q];
    uint32_t r = 0;
    if (dv[q] && s.window) {  // gamma(d) then unary(r)
      DevBits pk;
      pk.init_bit(s.words, rbit[r0 + k]);
      pk.gamma();
      r = pk.unary();
      if (r > k || r > s.window) {
        atomicExch(err, 1);
        r = 0;
      }
    }
    rr[k] = (uint8_t)r;
    if (ref_out && k < nr) ref_out[r0 + k] = (uint8_t)r;  // the rows' reference distances (device layout build)
    dep[k] = r ? 0xffffu : 0u;
    lvl[k] = 0;
  }
  if (t < 2) lvl[T + t] = 0;
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += u;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  uint32_t pre = inc - sum;
  for (uint32_t q = 0; q < w; ++q) pre += wsum[q];
#pragma unroll
  for (uint32_t q = 0; q < RPT; ++q) {
    loff[k0 + q] = pre;
    pre += dv[q];
  }
  if (k0 + RPT == T) loff[T] = pre;
  // depths: one barrier-separated sweep per chain step (reads of a sweep see
  // the previous sweep's writes only)
  for (uint32_t sweep = 0;; ++sweep) {
    int open = 0;
    uint16_t nd[RPT];
#pragma unroll
    for (uint32_t q = 0; q < RPT; ++q) {
      const uint32_t k = k0 + q;
      nd[q] = dep[k];
      if (nd[q] == 0xffffu) {
        const uint16_t pd = dep[k - rr[k]];
        if (pd != 0xffffu) nd[q] = (uint16_t)(pd + 1);
        else open = 1;
      }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t q = 0; q < RPT; ++q) dep[k0 + q] = nd[q];
    if (!__syncthreads_or(open)) break;
    if (sweep > T) {
      if (t == 0) atomicExch(err, 14);
      return;
    }
  }
  // counting sort by depth
  for (uint32_t k = t; k < nr; k += kDecThreads) atomicAdd(&lvl[dep[k]], 1u);
  __syncthreads();
  if (w == 0) {  // exclusive scan of the level counts (rows of the tile's padding have depth 0 and are not counted)
    uint32_t carry = 0, L = 0;
    for (uint32_t b0 = 0; b0 < T + 1; b0 += 32) {
      const uint32_t c = b0 + lane < T + 1 ? lvl[b0 + lane] : 0u;
      uint32_t iv = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, iv, o);
        if (lane >= (uint32_t)o) iv += u;
      }
      if (b0 + lane < T + 1) lvl[b0 + lane] = carry + iv - c;
      const uint32_t nz = __ballot_sync(0xffffffffu, c != 0);
      if (nz) L = b0 + 32 - __clz(nz);
      carry += __shfl_sync(0xffffffffu, iv, 31);
    }
    if (lane == 0) {
      nlev = L;
      lvl[T + 1] = carry;
    }
  }
  __syncthreads();
  for (uint32_t k = t; k < nr; k += kDecThreads) {
    const uint32_t at = atomicAdd(&lvl[dep[k]], 1u);  // lvl[d] becomes the end of level d
    order[at] = (uint16_t)k;
  }
  __syncthreads();
  const uint32_t total = loff[nr];
  const bool staged = total <= cap;
  uint32_t* outb = staged ? buf : cols + base;
  for (uint32_t k = t; k < nr; k += kDecThreads) row_offsets[r0 + k] = base + loff[k];
  if (r0 + nr == s.n && t == 0) row_offsets[s.n] = base + total;
  const uint32_t L = nlev;
  constexpr uint32_t NW = kDecThreads / 32;
  for (uint32_t d = 0; d < L; ++d) {
    const uint32_t beg = d ? lvl[d - 1] : 0u, end = lvl[d];
    // batches of 32 rows per warp; the lanes step their rows together
    for (uint32_t b0 = beg + 32 * w; b0 < end; b0 += 32 * NW) {
      const uint32_t idx = b0 + lane;
      RowDec rd;
      bool live = false;
      uint32_t i = 0;
      if (idx < end) {
        const uint32_t k = order[idx];
        i = r0 + k;
        const uint32_t r = rr[k];
        const uint32_t* Rl = r ? outb + loff[k - r] : nullptr;
        const uint32_t drl = r ? loff[k - r + 1] - loff[k - r] : 0u;
        live = rd.init(s, i, rbit[i], deg[i], outb + loff[k], Rl, drl, err);
      }
      bool run = live && rd.more1();
      while (__any_sync(0xffffffffu, run)) {
        if (run) run = rd.step1(s.n, err) && rd.more1();
      }
      if (live) rd.start2();
      run = live && rd.more2();
      while (__any_sync(0xffffffffu, run)) {
        if (run) run = rd.step2(s.n, err) && rd.more2();
      }
      if (live) rd.finish(s, i + 1 < s.n ? rbit[i + 1] : s.seg_bits[s.nseg], err);
    }
    __syncthreads();  // level d written before level d + 1 reads it
  }
  if (staged) {
    for (uint32_t e = t; e < total; e += kDecThreads) cols[base + e] = buf[e];
  }
}

}  // namespace cmvg
