// BV-D: the device layout of a BV-compressed matrix (shared by the host
// builder and the CUDA kernels; plain types only).
//
// It stores per row i the reference's differential row (cmv::ReferencedMatrix,
// reference include/cmv/ref_matrix.hpp:13-52) taken from the
// BV stream: the BV reference distance r, the minus entries (the reference
// entries that BV's copy blocks skip) and BV's extra list split exactly as BV
// splits it, into intervals and residuals.  The product is
//     y_i = y_{i-r} - sum_minus x + sum_intervals x + sum_residuals x
// (ref_matvec.hpp:20-31), an interval in O(1) from a prefix of x.
//
// The layout is built for the decoder's instruction budget, not for bits (the
// product is issue-bound, far from the HBM roofline): every code is a
// fixed-width field whose bit offset is known from the row header, so codes
// decode independently and rows can be processed in any order.
//
// Rows are grouped in blocks of `block_rows` (a multiple of the BV segment,
// so reference chains never leave a block).  A block's stream is
//   [row headers: block_rows x u32][row bodies, bit-packed, row order]  (16-B padded)
// Row header (u32, MSB first):
//   r (3) | #minus (5, 31 = escape) | #residual (6, 63 = escape) |
//   #interval (4, 15 = escape) | wp (5) | wl (5) | far (1) | 0 (3)
// (escaped rows keep their real counts in an escape table after the headers:
// entries (row, #minus, #residual, #interval)).
// Row body (bits):
//   [#minus + #residual point codes, wp bits each: col - i + bias]
//   [#interval x (left - i + bias in wp bits, len - Lmin in wl bits)]
// with bias = 2^(wp-1) (0 when wp = 0).  `far` marks rows with a column
// outside the block's x-window; only those rows take the bounds-checked path.  The
// row body length follows from the header, so the kernel computes every
// row's bit offset with one scan.
// Each block also carries an x-window start: the CTA stages x[wlo, wlo + W)
// (plus a tile-local prefix) in shared memory.
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#define __device__
#endif
#endif

namespace cmvg {

constexpr uint32_t kHdrMinusEsc = 31;
constexpr uint32_t kHdrResEsc = 63;
constexpr uint32_t kHdrIntEsc = 15;

__host__ __device__ constexpr uint32_t hdr_r(uint32_t h) { return h >> 29; }
__host__ __device__ constexpr uint32_t hdr_nm(uint32_t h) { return (h >> 24) & 31u; }
__host__ __device__ constexpr uint32_t hdr_ns(uint32_t h) { return (h >> 18) & 63u; }
__host__ __device__ constexpr uint32_t hdr_ni(uint32_t h) { return (h >> 14) & 15u; }
__host__ __device__ constexpr uint32_t hdr_wp(uint32_t h) { return (h >> 9) & 31u; }
__host__ __device__ constexpr uint32_t hdr_wl(uint32_t h) { return (h >> 4) & 31u; }
__host__ __device__ constexpr bool hdr_far(uint32_t h) { return (h >> 3) & 1u; }
__host__ __device__ constexpr uint32_t code_bias(uint32_t wp) { return wp ? (1u << (wp - 1)) : 0u; }
__host__ __device__ constexpr bool hdr_escaped(uint32_t h) {
  return hdr_nm(h) == kHdrMinusEsc || hdr_ns(h) == kHdrResEsc || hdr_ni(h) == kHdrIntEsc;
}
__host__ __device__ constexpr uint32_t make_hdr(uint32_t r, uint32_t nm, uint32_t ns, uint32_t ni, uint32_t wp,
                                                uint32_t wl, bool far) {
  return (r << 29) | (nm << 24) | (ns << 18) | (ni << 14) | (wp << 9) | (wl << 4) | ((far ? 1u : 0u) << 3);
}

// ---------------------------------------------------------------------------
// BV-S: the sliced variant used by the gather / PageRank kernels.  The same
// differential rows as BV-D (minus entries, residuals, intervals against the
// BV reference), re-cut by the transcoder into the kernel's work schedule:
//   * every light row is split into units of <= kBvsUnitPts point codes
//     (minus first, then residuals) and <= kBvsUnitInts intervals;
//   * per block, units are sorted by (code class, far, #intervals, #points)
//     and dealt into 32-lane slices, so a warp decodes 32 units of near-equal
//     work (lane utilisation ~85-95% instead of ~60% for whole rows);
//   * codes are byte aligned and relative to the block's x-window start wlo
//     (so a unit decodes without its row index).  Near class-16 slices (every
//     column inside the window -- the common case) are rectangular: each lane
//     holds ceil(max #points / 2) point words, two 16-bit codes each (first
//     in the high half), code = padded window index | minus << 15, lanes with
//     fewer points padded with the window's zero entry; then max #intervals
//     words (left - wlo) << 16 | len (0 = empty).  Far class-16 units store
//     16-bit codes col - wlo + 2^15 (two per word) and intervals
//     (left - wlo + 2^15) << 16 | (len - Lmin), per lane counts from the
//     header; class 32
//     stores absolute columns, one word per point, two per interval
//     (left, len - Lmin).  A slice's lane streams are interleaved: word q of
//     lane l at body + 32 q + l (one conflict-free shared load per word);
//   * a row that needs 2..32 units puts them in adjacent lanes of one
//     "multi" slice (rows packed first-fit decreasing); the warp combines a
//     row's lanes with a segmented shuffle reduction and the row's first
//     unit (its primary) writes delta_i and r_i.  Rows needing more than 32
//     units are decoded by a whole warp from a row-major, bit-packed heavy
//     stream (BV-D codes).
// Block stream (u32 words):
//   [0] nslices | nheavy << 16   [1] heavy table offset   [2] heavy stream offset
//   [3] the block's first heavy-row work item (global numbering: the
//   partial-sum slot of its chunk 0)   [4, 9) u16 start of warp w's slices in the table (w < 8), then
//   the table size: the static warp schedule (longest-processing-time
//   assignment by an instruction estimate; warp w decodes entries
//   [start_w, start_{w+1}))   [9] 0
//   [10, 10 + 2 nslices) slice table: (record offset, meta) per slice
//   slice record: [meta][header x 32][body]
//     meta: max #points | max #intervals << 5 | class32 << 8 | far << 9 |
//           multi << 10
//     header: valid << 31 | primary << 30 | k << 20 | r << 17 |
//             #minus << 12 | #points << 7 | #intervals << 4
//   heavy table: kBvsHeavyEntry words per heavy row: BV-D-style a-word
//     (make_sa), #minus, #residual, #interval, bit offset in the heavy stream,
//     first work item of the row within the block (a heavy row's points are
//     cut into heavy_chunks(#points) items of kBvsHeavyChunk, decoded by any
//     warp; their partial sums are combined in item order)
//   heavy stream: the heavy rows' BV-D bodies, bit-packed, MSB first
#ifndef CMVG_UNIT_PTS  // build-time override for A/B experiments (<= 31: the 5-bit count fields)
#define CMVG_UNIT_PTS 16
#endif
constexpr uint32_t kBvsUnitPts = CMVG_UNIT_PTS;
constexpr uint32_t kBvsUnitInts = 2;
constexpr uint32_t kBvsMaxUnits = 32;  // more -> heavy row
constexpr uint32_t kBvsHeavyEntry = 6;
constexpr uint32_t kBvsHeavyChunk = 512;  // points per work item of a heavy row (16 per lane)
__host__ __device__ constexpr uint32_t heavy_chunks(uint32_t np) {
  return np > kBvsHeavyChunk ? (np + kBvsHeavyChunk - 1) / kBvsHeavyChunk : 1u;
}
constexpr uint32_t kBvsWarps = 8;     // warps of the gather CTA the static schedule is built for
constexpr uint32_t kBvsWarpTab = 4;   // header words [4, 9): u16 slice-table start per warp, + end
constexpr uint32_t kBvsHead = 10;
constexpr uint32_t kBvsBias16 = 32768;
// padded x-window index (8-entry tiles at a stride of 9; cuda/xwindow.cuh)
__host__ __device__ constexpr uint32_t bvs_pad_index(uint32_t j) { return j + (j >> 3); }
__host__ __device__ constexpr uint32_t make_sa(uint32_t k, uint32_t r, uint32_t wp, uint32_t wl, bool far) {
  return k | (r << 12) | (wp << 15) | (wl << 20) | ((far ? 1u : 0u) << 25) | (1u << 31);
}
__host__ __device__ constexpr uint32_t sa_k(uint32_t a) { return a & 4095u; }
__host__ __device__ constexpr uint32_t sa_r(uint32_t a) { return (a >> 12) & 7u; }
__host__ __device__ constexpr uint32_t sa_wp(uint32_t a) { return (a >> 15) & 31u; }
__host__ __device__ constexpr uint32_t sa_wl(uint32_t a) { return (a >> 20) & 31u; }
__host__ __device__ constexpr bool sa_far(uint32_t a) { return (a >> 25) & 1u; }

__host__ __device__ constexpr uint32_t make_uh(bool primary, uint32_t k, uint32_t r, uint32_t nm, uint32_t np,
                                               uint32_t ni) {
  return (1u << 31) | ((primary ? 1u : 0u) << 30) | (k << 20) | (r << 17) | (nm << 12) | (np << 7) | (ni << 4);
}
__host__ __device__ constexpr bool uh_valid(uint32_t h) { return h >> 31; }
__host__ __device__ constexpr bool uh_primary(uint32_t h) { return (h >> 30) & 1u; }
__host__ __device__ constexpr uint32_t uh_k(uint32_t h) { return (h >> 20) & 1023u; }
__host__ __device__ constexpr uint32_t uh_r(uint32_t h) { return (h >> 17) & 7u; }
__host__ __device__ constexpr uint32_t uh_nm(uint32_t h) { return (h >> 12) & 31u; }
__host__ __device__ constexpr uint32_t uh_np(uint32_t h) { return (h >> 7) & 31u; }
__host__ __device__ constexpr uint32_t uh_ni(uint32_t h) { return (h >> 4) & 7u; }
// rounds: shuffle rounds of a multi slice's segmented reduction,
// ceil(log2(max units of one row in the slice)) (0 for single-unit slices)
__host__ __device__ constexpr uint32_t make_smeta(uint32_t max_np, uint32_t max_ni, bool c32, bool far, bool multi,
                                                  uint32_t rounds = 0) {
  return max_np | (max_ni << 5) | ((c32 ? 1u : 0u) << 8) | ((far ? 1u : 0u) << 9) | ((multi ? 1u : 0u) << 10) |
         (rounds << 11);
}
__host__ __device__ constexpr uint32_t smeta_np(uint32_t m) { return m & 31u; }
__host__ __device__ constexpr uint32_t smeta_ni(uint32_t m) { return (m >> 5) & 7u; }
__host__ __device__ constexpr bool smeta_c32(uint32_t m) { return (m >> 8) & 1u; }
__host__ __device__ constexpr bool smeta_far(uint32_t m) { return (m >> 9) & 1u; }
__host__ __device__ constexpr bool smeta_multi(uint32_t m) { return (m >> 10) & 1u; }
__host__ __device__ constexpr uint32_t smeta_rounds(uint32_t m) { return (m >> 11) & 7u; }

// ---------------------------------------------------------------------------
// BV-T: the scatter form's stream (y = x A on A's own compression).  Per block
// the transcoder groups A's differential contributions by TARGET column: row
// k contributes -c_k at each minus column, +c_k at each residual column, and
// an interval [a, a + len) becomes two difference entries (+c_k at a, -c_k at
// a + len) whose running sum covers the run, where c_k = x_k + sum of c over
// the rows that reference k (Proposition 1 applied to x A).  A target's
// segment is then summed with the gather's slice machinery -- no atomics:
//   targets t < W            point sums at window column wlo + t
//           W <= t < 2W      difference entries at window column wlo + t - W
//           2W <= t          far column far[t - 2W] (outside the window)
//   codes: 16-bit k | minus << 15 (k = block row; k = B reads a zero
//          coefficient -- the padding code), two per word, rectangular slices
// Block stream (u32 words):
//   [0] nslices | nheavy << 16  [1] heavy table offset  [2] heavy code offset
//   [3] nfar  [4] coefficient schedule offset  [5] far column list offset
//   [6, 7] 0  [8, 8 + 2 nslices) slice table: (record offset, meta) per slice
//   coefficient schedule: [nlev][nlev + 1 level starts][entries]; levels
//     deepest first, entry = k | children mask << 10 (bit r-1: row k + r
//     references k), rows without children omitted
//   far list: nfar absolute columns, ascending
//   slice record: [meta][header x 32][body: ceil(max entries / 2) words x 32]
//     meta: max entries | multi << 10
//     header: valid << 31 | primary << 30 | target
//   heavy table: 3 words per heavy target: target, #entries, code word offset
//   heavy codes: 16-bit codes, two per word
// Block table entry: word_offset, nwords, wlo as BV-D; pad[0] = first far
// staging slot of the block.
constexpr uint32_t kBvtHead = 8;
constexpr uint32_t kBvtUnitCodes = 16;  // codes per target unit
constexpr uint32_t kBvtMaxUnits = 32;   // units of a slice target (more: heavy target)
constexpr uint32_t kBvtHeavyEntry = 3;
__host__ __device__ constexpr uint32_t make_th(bool primary, uint32_t target) {
  return (1u << 31) | ((primary ? 1u : 0u) << 30) | target;
}
__host__ __device__ constexpr uint32_t th_target(uint32_t h) { return h & 0x3fffffffu; }
// rounds: as smeta_rounds (segmented-reduction rounds of a multi slice)
__host__ __device__ constexpr uint32_t make_tmeta(uint32_t max_ne, bool multi, uint32_t rounds = 0) {
  return max_ne | ((multi ? 1u : 0u) << 10) | (rounds << 11);
}
__host__ __device__ constexpr uint32_t tmeta_ne(uint32_t m) { return m & 1023u; }
__host__ __device__ constexpr bool tmeta_multi(uint32_t m) { return (m >> 10) & 1u; }
__host__ __device__ constexpr uint32_t tmeta_rounds(uint32_t m) { return (m >> 11) & 7u; }

// ---------------------------------------------------------------------------
// BV-F: the flat term stream of the gather / PageRank kernels
// (cuda/bvf_gather.cuh).  The same differential rows as BV-D (reference
// include/cmv/ref_matrix.hpp:13-52; y_i = y_{i-r} - sum_minus x + sum_plus x,
// ref_matvec.hpp:20-31), written as one flat list of 16-bit TERMS per block in
// row order.  A term is one signed entry of a per-block shared-memory table:
//   table[0, W)                x[wlo + j]            (the block's x-window)
//   table[W, W + nslot)        x[far[s]]             (columns outside the window)
//   table[W + kBvfSlots]       0                     (padding / empty rows)
//   table[F0 + j], j <= W      F[j] = sum_{t < j} x[wlo + t]   (F0 = W + kBvfSlots + 1)
// so a minus entry is -x[c], a residual +x[c] and an interval [a, a + len)
// inside the window the two terms +F[a - wlo + len], -F[a - wlo] (O(1),
// PAPER.md:198-206).  Intervals reaching outside the window are written as
// their columns.  Term (16 bits): index (13) | escape << 13 | end << 14 |
// minus << 15; `end` marks a row's last term (every row has an even number
// >= 2 of terms, padded with zero-entry terms, so a row ends only on the
// second (high) term of a code word).  Escape terms (blocks whose far columns
// exceed the slots) read x[esc[escstart_t + index]] from global memory.
// Work split: the block's N terms are cut into nact chunks of K terms
// (K = 16 ceil(N / 4096), nact = ceil(N / K) <= 256; the last chunk padded);
// thread t sums chunk t, so every thread has the same work whatever the row
// lengths (hub rows need no special path); a row cut by a chunk boundary is
// completed by the next thread that ends it (carry).
// Block stream (u32 words):
//   [0, align4(ceil(nact/2)))   u16 first row of each chunk
//   [.., + kBvfRnWords)         reference distance r of each row, 4 bits (8 per word)
//   [.., + align4(nslot))       far slot columns
//   esc_off: (escape blocks) u32 first escape of each chunk and the total
//                            [align4(nact + 1)], then the escape columns
//                            [align4(nesc)], the 32 chunks of a warp interleaved
//                            (by term position, then lane: bvf_block.hpp)
//   codes_off: K/2 x nact words, word q of chunk t at codes_off + q nact + t
//     (two terms per word, the first in the low half: coalesced loads)
constexpr uint32_t kBvfSlots = 127;    // far slots per block (the next entry is the zero entry; odd: F0 even)
constexpr uint32_t kBvfMaxThreads = 256;
constexpr uint32_t kBvfRnWords = 128;  // 1024 rows x 4 bits
constexpr uint32_t kBvfIdxMask = 0x1fffu;
constexpr uint32_t kBvfEsc = 0x2000u, kBvfEnd = 0x4000u, kBvfMinus = 0x8000u;
constexpr uint32_t kBvfFlagEsc = 1u;  // BvfBlockInfo::flags: the block has escape terms
__host__ __device__ constexpr uint32_t bvf_f0(uint32_t W) { return W + kBvfSlots + 1; }
__host__ __device__ constexpr uint32_t bvf_zero(uint32_t W) { return W + kBvfSlots; }
__host__ __device__ constexpr uint32_t bvf_align4(uint32_t v) { return (v + 3u) & ~3u; }
__host__ __device__ constexpr uint32_t bvf_rn_off(uint32_t nact) { return bvf_align4((nact + 1u) / 2u); }
__host__ __device__ constexpr uint32_t bvf_far_off(uint32_t nact) { return bvf_rn_off(nact) + kBvfRnWords; }

struct BvfBlockInfo {
  uint64_t word_offset;  // first u32 word of the block's stream (16-byte aligned)
  uint32_t wlo;          // x-window start
  uint16_t K, nact;      // terms per chunk, chunks (active threads)
  uint16_t nslot;        // far slots used
  uint8_t cbits;         // grid of the exact split: G = 2^(E - cbits), E = block max exponent
  uint8_t flags;
  uint32_t codes_off;    // word offset of the term words
  uint32_t esc_off;      // word offset of the escape tables (escape blocks)
  uint32_t nwords;
};
static_assert(sizeof(BvfBlockInfo) == 32, "BvfBlockInfo is 32 bytes");

struct BvdBlockInfo {
  uint64_t word_offset;  // first u32 word of this block's stream (16-byte aligned)
  uint32_t nwords;       // words in this block's stream (multiple of 4)
  uint32_t wlo;          // x-window start (multiple of 16)
  uint32_t nesc;         // escaped rows (entries of the escape table)
  uint32_t pad[3];
};

struct BvdDims {
  uint32_t n;            // rows (== columns)
  uint32_t block_rows;   // B
  uint32_t window;       // x-window entries (multiple of 16)
  uint32_t min_interval;
  uint32_t nblocks;
  uint32_t max_block_words;
  uint32_t max_depth;    // longest reference chain (drives the level phases)
  uint32_t pad;
};

}  // namespace cmvg
