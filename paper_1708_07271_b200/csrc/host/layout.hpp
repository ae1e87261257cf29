// BV-D: the device layout of a BV-compressed matrix (shared by the host
// builder and the CUDA kernels; plain types only).
//
// What it stores (per row i, in row order) is the reference's differential
// row (cmv::ReferencedMatrix, reference include/cmv/ref_matrix.hpp:13-52 and
// PAPER.md:156-196) with BV's codes:
//   bits(ref_bits)  r: reference distance, 0 = self-coded
//   if r > 0:       gamma(#minus); minus columns = the reference entries that
//                   BV's copy blocks skip, zeta_k gap-coded (first sign-folded
//                   relative to i, then gap-1)
//   gamma(#intervals); intervals exactly as in the BV stream
//   gamma(#residuals); residuals exactly as in the BV stream
// so the product is  y_i = y_{i-r} - sum_minus x + sum_intervals x (O(1) from
// an exclusive prefix of x) + sum_residuals x  (ref_matvec.hpp:20-31).
//
// Rows are grouped in blocks of `block_rows` (a multiple of the BV segment, so
// reference chains never leave a block).  Each block's stream is split into
// `lanes` contiguous row ranges with balanced decode cost; lane k's bits start
// byte-aligned and the lane table entry packs (byte offset << row_bits) |
// first row.  Each block also carries an x-window start: the CTA stages
// x[wlo, wlo + window) (plus a tile-local prefix) in shared memory.
#pragma once
#include <cstdint>

namespace cmvg {

struct BvdBlockInfo {
  uint64_t word_offset;  // first u32 word of this block's stream (16-byte aligned)
  uint32_t nwords;       // words in this block's stream (multiple of 4)
  uint32_t wlo;          // x-window start (multiple of 16)
};

struct BvdDims {
  uint32_t n;            // rows (== columns)
  uint32_t block_rows;   // B
  uint32_t lanes;        // T (decode lanes per block = threads per CTA)
  uint32_t row_bits;     // width of the row field in a lane entry (log2(B)+1)
  uint32_t window;       // x-window entries (multiple of 16)
  uint32_t ref_bits;     // bits of the reference-distance field
  uint32_t min_interval;
  uint32_t zeta_k;
  uint32_t nblocks;
  uint32_t max_block_words;
  uint32_t max_depth;    // longest reference chain (drives the level phases)
  uint32_t pad;
};

}  // namespace cmvg
