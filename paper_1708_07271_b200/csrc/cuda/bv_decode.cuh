// bv_decode_csr: canonical BV stream -> CSR on the device, bit-exact with the
// source adjacency (the GPU counterpart of `reconstruct_graph`,
// reference include/cmv/ref_matrix.hpp:75-76, with BV copy blocks resolved
// positionally against the decoded reference list).
//
// Segments are chain-closed, so one thread decodes one segment serially:
//   pass 1 (bv_seg_degrees): parse only, write out-degrees + segment edge sums;
//   host/device scan of segment sums;
//   pass 2 (bv_seg_decode): write row offsets and columns; a row's copied
//      entries are read back from its reference row's freshly written output
//      and merged with its intervals and residuals (three lazy cursors).
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
  PosBits br{s.words, s.seg_bits[sg]};
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
      copied = bv_skip_blocks(br, deg[i - r]);
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
      for (uint64_t k = in_int; k < extra; ++k) br.zeta(s.zeta_k);
    }
  }
  if (br.pos != s.seg_bits[sg + 1]) atomicExch(err, 4);
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
    uint64_t d = br.gamma();
    if (d == 0) continue;
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
    // interval state
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
    // residual state
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
      if (v >= s.n || (written && v <= prev) || written >= d) { atomicExch(err, 5); return; }
      cols[off + written] = (uint32_t)v;
      prev = (uint32_t)v;
      ++written;
    }
    if (written != d) { atomicExch(err, 6); return; }
    off += d;
  }
  if (br.pos != s.seg_bits[sg + 1]) atomicExch(err, 7);
  if (sg == s.nseg - 1) row_offsets[s.n] = off;
}

}  // namespace cmvg
