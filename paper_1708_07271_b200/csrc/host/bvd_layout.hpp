#pragma once
#include <vector>

#include "host.hpp"
#include "layout.hpp"

namespace cmvg {

struct BvdOptions {
  uint32_t block_rows = 1024;
  uint32_t window = 2048;
  bool bvs = true;  // build the sliced layout (matmat)
  bool bvt = true;  // build the target-sorted layout (scatter)
  bool bvf = true;  // build the flat term layout (gather / PageRank)
};

struct BvdStats {
  uint64_t row_bits = 0;          // sum of row-record bits (the coded payload)
  uint64_t stream_bytes = 0;      // incl. lane alignment and block padding
  uint64_t block_table_bytes = 0;
  uint64_t codes = 0;             // body codes (decode loop iterations)
  uint32_t p995_block_words = 0;  // block-stream size covering 99.5% of blocks
  double window_coverage = 1.0;   // fraction of gathered columns inside the x-window
};

struct BvsStats {
  uint64_t stream_bytes = 0;
  uint32_t max_block_words = 0;
  uint32_t p995_block_words = 0;
  uint64_t slices = 0, heavy_rows = 0;
  uint64_t heavy_chunks = 0;                      // work items of the heavy rows (kBvsHeavyChunk points each)
  uint64_t lane_words = 0, lane_words_used = 0;  // slice body words incl. / excl. padding
  uint64_t lane_iters = 0, lane_iters_used = 0;  // slice decode iterations x 32 / useful lane iterations
};

struct BvfStats {
  uint64_t stream_bytes = 0;
  uint64_t terms = 0;         // useful terms (x entries, interval ends, refs not counted)
  uint64_t pad_terms = 0;     // padding terms (empty rows, chunk tails)
  uint64_t slot_terms = 0;    // terms on far slots
  uint64_t esc_terms = 0;     // terms read from global memory (slots exhausted)
  uint64_t esc_blocks = 0;
  uint32_t max_K = 0;
  uint32_t min_cbits = 64;
};

struct BvtStats {
  uint64_t stream_bytes = 0;
  uint64_t slices = 0, heavy_targets = 0, far_slots = 0, entries = 0;
  uint64_t lane_iters = 0, lane_iters_used = 0;
};

struct BvdLayout {
  BvdDims dims{};
  std::vector<uint32_t> words;
  std::vector<BvdBlockInfo> blocks;
  // BV-S (sliced) stream of the same blocks; same block table fields, same wlo
  std::vector<uint32_t> swords;
  std::vector<BvdBlockInfo> sblocks;
  BvsStats sstats;
  // BV-F (flat term stream; gather / PageRank)
  std::vector<uint32_t> fwords;
  std::vector<BvfBlockInfo> fblocks;
  BvfStats fstats;
  // BV-T (target-sorted scatter stream) + the combine tables
  std::vector<uint32_t> twords;
  std::vector<BvdBlockInfo> tblocks;  // pad[0] = first far staging slot
  BvtStats tstats;
  std::vector<uint32_t> tile_ptr, tile_blk;  // per 'block_rows' column tile: blocks whose window meets it
  std::vector<uint32_t> farp_ptr;            // per tile: range in farp
  std::vector<uint32_t> farp;                // (column, far slot) pairs sorted by column
  // columns each block reads outside its x-window, sorted (CSR by block)
  std::vector<uint64_t> rfar_ptr;
  std::vector<uint32_t> rfar;
  uint64_t adds_per_product = 0;
  BvdStats stats;
};

BvdLayout build_bvd(const BvDecoded& dec, const BvParams& bp, const BvdOptions& opt);

}  // namespace cmvg
