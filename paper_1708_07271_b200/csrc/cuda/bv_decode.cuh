// bv_decode_csr: canonical BV stream -> CSR on the device, bit-exact with the
// source adjacency (the GPU counterpart of `reconstruct_graph`,
// reference include/cmv/ref_matrix.hpp:75-76, with BV copy blocks resolved
// positionally against the decoded reference list).
//
// Segments are chain-closed, so they decode independently:
//   pass 1 (bv_seg_degrees, one thread per segment): parse only, write
//      out-degrees + segment edge sums; host scan of the segment sums;
//   pass 2 (bv_seg_decode_warp, one warp per segment): write row offsets and
//      columns; a row's copied entries are read back from its reference row's
//      freshly written output and merged with its intervals and residuals
//      (see below).  bv_seg_decode is the serial (thread-per-segment) form.
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

__global__ void bv_seg_degrees(BvDev s, uint32_t* __restrict__ deg, uint64_t* __restrict__ seg_edges,
                               int* __restrict__ err) {
  uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x;
  if (sg >= s.nseg) return;
  uint32_t r0 = sg * s.seg_rows;
  uint32_t r1 = min(s.n, r0 + s.seg_rows);
  DevBits br;  // register window: one 32-bit load per 32 bits parsed
  br.init_bit(s.words, s.seg_bits[sg]);
  uint64_t tot = 0;
  for (uint32_t i = r0; i < r1; ++i) {
    uint64_t d = br.gamma();
    deg[i] = (uint32_t)d;
    tot += d;
    if (d == 0) continue;
    uint32_t r = s.window ? br.unary() : 0u;
    uint64_t copied = 0;
    if (r) {
      if (r > s.window || i < r0 + r) { atomicExch(err, 1); return; }
      const uint64_t dr = deg[i - r];
      const uint64_t b = br.gamma();
      uint64_t pos = 0;
      bool cp = true;
      for (uint64_t k = 0; k < b; ++k) {
        const uint64_t len = k == 0 ? br.gamma() : br.gamma() + 1;
        if (cp) copied += len;
        pos += len;
        cp = !cp;
      }
      if (cp && dr > pos) copied += dr - pos;
    }
    if (copied > d) { atomicExch(err, 2); return; }
    uint64_t extra = d - copied;
    if (extra) {
      uint64_t ni = br.gamma(), in_int = 0;
      for (uint64_t k = 0; k < ni; ++k) {
        br.gamma();
        in_int += br.gamma() + s.min_interval;
      }
      if (in_int > extra) { atomicExch(err, 3); return; }
      for (uint64_t k = in_int; k < extra; ++k) br.zeta<3>();
    }
  }
  if (br.bitpos(s.words) != s.seg_bits[sg + 1]) atomicExch(err, 4);
  seg_edges[sg] = tot;
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
  if (sg >= s.nseg) return;
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
// Warp-cooperative decoder: one warp per segment.  Lane 0 parses a row's
// instantaneous codes (gamma out-degree, unary reference, gamma copy-block
// lengths, gamma interval gaps / lengths, zeta_k residual gaps -- inherently
// sequential) into per-warp shared-memory lists; then the whole warp
//   * selects the copied entries of the reference row (each lane tests its
//     positions against the block boundaries -- binary search -- and a ballot
//     prefix compacts them),
//   * expands the intervals, and
//   * merges the three sorted, disjoint lists by rank (each element's output
//     position = its index + the number of smaller elements in the other two
//     lists, by binary search), writing the row's columns in parallel.
// Rows whose lists exceed the per-warp buffers fall back to the serial row
// decoder on lane 0.
constexpr uint32_t kDecBlocks = 128, kDecInts = 64, kDecRes = 512, kDecCopy = 1024;
struct DecWarpSmem {
  uint32_t blk[kDecBlocks];      // copy-block boundaries (run ends) in the reference list
  uint32_t ileft[kDecInts], ipre[kDecInts + 1];
  uint32_t res[kDecRes];
  uint32_t cpy[kDecCopy];
};

// number of entries < x in the sorted list v[0, n)
__device__ __forceinline__ uint32_t dec_count_less(const uint32_t* v, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (v[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// number of interval elements < x (intervals sorted, disjoint; ipre exclusive prefix of lengths)
__device__ __forceinline__ uint32_t dec_count_less_int(const DecWarpSmem& w, uint32_t ni, uint32_t x) {
  const uint32_t u = dec_count_less(w.ileft, ni, x);  // intervals starting below x
  if (u == 0) return 0;
  const uint32_t len = w.ipre[u] - w.ipre[u - 1];
  const uint32_t inside = min(len, x - w.ileft[u - 1]);
  return w.ipre[u - 1] + inside;
}

__global__ void __launch_bounds__(128) bv_seg_decode_warp(BvDev s, const uint64_t* __restrict__ seg_base,
                                                          uint64_t* __restrict__ row_offsets,
                                                          uint32_t* __restrict__ cols, int* __restrict__ err) {
  __shared__ DecWarpSmem sw[4];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const uint32_t sg = blockIdx.x * 4u + wid;
  if (sg >= s.nseg) return;
  DecWarpSmem& w = sw[wid];
  const uint32_t r0 = sg * s.seg_rows, r1 = min(s.n, r0 + s.seg_rows);
  DevBits br;  // lane 0's cursor: a 64-bit register window, one load per 32 bits
  if (lane == 0) br.init_bit(s.words, s.seg_bits[sg]);
  uint64_t off = seg_base[sg];
  for (uint32_t i = r0; i < r1; ++i) {
    // ---- lane 0: parse the row's codes into the per-warp lists ----
    uint32_t d = 0, r = 0, nblk = 0, ni = 0, nres = 0, in_int = 0, fb = 0;
    uint64_t row_start = lane == 0 ? br.bitpos(s.words) : 0;
    if (lane == 0) {
      row_offsets[i] = off;
      d = (uint32_t)br.gamma();
      if (d) {
        r = s.window ? br.unary() : 0u;
        uint64_t copied = 0;
        if (r) {
          const uint32_t dr = (uint32_t)(row_offsets[i - r + 1] - row_offsets[i - r]);
          const uint32_t b = (uint32_t)br.gamma();
          uint32_t pos = 0;
          bool cp = true;
          for (uint32_t k = 0; k < b; ++k) {
            const uint32_t len = (uint32_t)(k == 0 ? br.gamma() : br.gamma() + 1);
            if (cp) copied += len;
            pos += len;
            if (k < kDecBlocks) w.blk[k] = pos;
            cp = !cp;
          }
          if (cp && dr > pos) copied += dr - pos;
          nblk = b;
          if (b > kDecBlocks || copied > kDecCopy) fb = 1;
        }
        const uint32_t extra = d - (uint32_t)copied;
        if (extra) {
          ni = (uint32_t)br.gamma();
          uint32_t prev_end = 0;
          w.ipre[0] = 0;
          for (uint32_t k = 0; k < ni; ++k) {
            const uint32_t left = k == 0 ? (uint32_t)((int64_t)i + unfold_i32((uint32_t)br.gamma()))
                                         : prev_end + (uint32_t)br.gamma() + 1u;
            const uint32_t len = (uint32_t)br.gamma() + s.min_interval;
            if (k < kDecInts) {
              w.ileft[k] = left;
              w.ipre[k + 1] = w.ipre[k] + len;
            }
            prev_end = left + len;
            in_int += len;
          }
          if (ni > kDecInts) fb = 1;
          nres = extra - in_int;
          int64_t v = 0;
          for (uint32_t k = 0; k < nres; ++k) {
            v = k == 0 ? (int64_t)i + unfold_i32(br.zeta<3>()) : v + (int64_t)br.zeta<3>() + 1;
            if (k < kDecRes) w.res[k] = (uint32_t)v;
          }
          if (nres > kDecRes) fb = 1;
        }
      }
    }
    d = __shfl_sync(0xffffffffu, d, 0);
    fb = __shfl_sync(0xffffffffu, fb, 0);
    if (fb) {  // oversized lists: serial row decode on lane 0 from the row start
      if (lane == 0) {
        PosBits rb{s.words, row_start};
        if (!bv_decode_row_serial(s, i, rb, off, row_offsets, cols, err)) atomicExch(err, 8);
        br.init_bit(s.words, rb.pos);
      }
      off += d;
      __syncwarp();
      continue;
    }
    if (d == 0) {
      __syncwarp();
      continue;
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    nblk = __shfl_sync(0xffffffffu, nblk, 0);
    ni = __shfl_sync(0xffffffffu, ni, 0);
    nres = __shfl_sync(0xffffffffu, nres, 0);
    in_int = __shfl_sync(0xffffffffu, in_int, 0);
    __syncwarp();  // lists in shared memory are complete
    // ---- copied entries of the reference row, compacted ----
    uint32_t nc = 0;
    if (r) {
      const uint64_t rb = row_offsets[i - r];
      const uint32_t dr = (uint32_t)(row_offsets[i - r + 1] - rb);
      for (uint32_t base = 0; base < dr; base += 32) {
        const uint32_t j = base + lane;
        bool take = false;
        uint32_t v = 0;
        if (j < dr) {
          const uint32_t t = nblk ? dec_count_less(w.blk, nblk, j + 1) : 0u;  // boundaries <= j
          take = (t & 1u) == 0;
          if (take) v = cols[rb + j];
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        if (take) w.cpy[nc + __popc(bal & ((1u << lane) - 1u))] = v;
        nc += __popc(bal);
      }
    }
    __syncwarp();
    if (lane == 0 && nc + in_int + nres != d) atomicExch(err, 9);
    // ---- rank merge of the three sorted lists ----
    uint32_t* out = cols + off;
    for (uint32_t a = lane; a < nc; a += 32) {
      const uint32_t x = w.cpy[a];
      out[a + dec_count_less_int(w, ni, x) + dec_count_less(w.res, nres, x)] = x;
    }
    for (uint32_t e = lane; e < in_int; e += 32) {
      const uint32_t u = dec_count_less(w.ipre + 1, ni, e + 1);  // interval holding element e
      const uint32_t x = w.ileft[u] + (e - w.ipre[u]);
      out[e + dec_count_less(w.cpy, nc, x) + dec_count_less(w.res, nres, x)] = x;
    }
    for (uint32_t a = lane; a < nres; a += 32) {
      const uint32_t x = w.res[a];
      if (x >= s.n) atomicExch(err, 5);
      out[a + dec_count_less(w.cpy, nc, x) + dec_count_less_int(w, ni, x)] = x;
    }
    off += d;
    __syncwarp();  // the row's columns are visible to later rows referencing it
  }
  if (lane == 0) {
    if (br.bitpos(s.words) != s.seg_bits[sg + 1]) atomicExch(err, 7);
    if (sg == s.nseg - 1) row_offsets[s.n] = off;
  }
}

}  // namespace cmvg
