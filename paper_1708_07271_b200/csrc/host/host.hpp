// Host-side data structures shared by the generators, the BV codec and the
// device-layout builder.  Everything here is preprocessing (untimed); the hot
// path is the CUDA product in ../cuda.
#pragma once
#include <algorithm>
#include <atomic>
#include <exception>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace cmvg {

// CSR adjacency of a directed graph: the layout of cmv::CsrGraph
// (reference include/cmv/csr.hpp:16-36): u64 row offsets, u32 columns,
// strictly increasing within each row.
struct HostCsr {
  uint32_t n = 0;
  std::vector<uint64_t> row_offsets;  // n+1
  std::vector<uint32_t> cols;         // m
  uint64_t m() const { return cols.size(); }
  uint32_t deg(uint32_t u) const { return (uint32_t)(row_offsets[u + 1] - row_offsets[u]); }
  const uint32_t* row(uint32_t u) const { return cols.data() + row_offsets[u]; }
};

// BV encoding parameters (BASELINE.json configs: w=7, R=3 or unbounded,
// Lmin=4, zeta_3 residuals).  `segment_rows`: references never cross a
// multiple of segment_rows, so segments decode independently.
struct BvParams {
  uint32_t window = 7;         // w
  uint32_t max_ref = 3;        // R; 0 = unbounded chains
  uint32_t min_interval = 4;   // Lmin
  uint32_t zeta_k = 3;         // residual code
  uint32_t segment_rows = 1024;
};

struct BvStats {
  uint64_t stream_bits = 0;
  uint64_t rows_with_ref = 0;
  uint64_t copied_edges = 0;
  uint64_t interval_edges = 0;
  uint64_t intervals = 0;
  uint64_t residual_edges = 0;
  uint64_t minus_edges = 0;    // reference entries skipped by copy blocks
  uint32_t max_depth = 0;      // longest reference chain
};

// The canonical BV stream (the interchange format; S = stream_bits).
struct BvStream {
  uint32_t n = 0;
  uint64_t m = 0;
  BvParams params;
  std::vector<uint32_t> words;
  uint64_t nbits = 0;
  std::vector<uint64_t> segment_bit_offsets;  // nseg + 1
  std::vector<uint8_t> ref_dist;              // per row, 0 = no reference (encoder side info)
  BvStats stats;
};

// Decoded reference structure (per row: reference distance plus the row's
// adjacency), produced by the CPU BV decoder.
struct BvDecoded {
  HostCsr csr;
  std::vector<uint8_t> ref_dist;
};

// ---- parallel helper ------------------------------------------------------
inline unsigned host_threads() {
  unsigned t = std::thread::hardware_concurrency();
  return t ? t : 1;
}
inline void parallel_for(uint64_t n, const std::function<void(uint64_t, uint64_t)>& body,
                         unsigned threads = 0, uint64_t grain = 1) {
  if (!threads) threads = host_threads();
  if (n == 0) return;
  uint64_t chunks = std::min<uint64_t>(n, (uint64_t)threads * 8);
  if (threads == 1 || n <= grain) { body(0, n); return; }
  std::atomic<uint64_t> next{0};
  std::exception_ptr err;
  std::atomic<bool> failed{false};
  auto worker = [&]() {
    for (;;) {
      uint64_t c = next.fetch_add(1);
      if (c >= chunks || failed.load()) break;
      uint64_t b = n * c / chunks, e = n * (c + 1) / chunks;
      try {
        if (b < e) body(b, e);
      } catch (...) {
        bool expect = false;
        if (failed.compare_exchange_strong(expect, true)) err = std::current_exception();
        break;
      }
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// ---- generators (gen.cpp) -------------------------------------------------
struct CopyModelParams {
  uint32_t n = 1u << 20;
  double mean_degree = 12;
  double p_ref = 0.7;
  uint32_t ref_window = 7;
  double p_copy = 0.8;
  double gap_mean = 64;
  double p_run = 0.3;
  uint32_t run_min = 4, run_max = 16;
  uint32_t gen_segment = 65536;  // copy sources stay inside a generator segment
  uint64_t seed = 0x170807271ull;
  double lambda = 0;             // 0 = calibrate to mean_degree
};
struct SocialParams {
  uint32_t n = 1u << 25;
  double zipf_exponent = 2.1;
  uint32_t deg_min = 1, deg_max = 100000;
  double zipf_shift = 4.465;
  double p_community = 0.8;
  uint32_t community = 4096;
  double p_ref = 0.5;
  uint32_t ref_window = 7;
  double p_copy = 0.6;
  uint32_t gen_segment = 65536;
  uint64_t seed = 0x170807271ull + 4;
};
double calibrate_copy_model_lambda(const CopyModelParams& p);
HostCsr generate_copy_model(const CopyModelParams& p);
HostCsr generate_social(const SocialParams& p);

// ---- BV codec (bv_codec.cpp) ----------------------------------------------
BvStream bv_encode(const HostCsr& g, const BvParams& p);
BvDecoded bv_decode(const BvStream& s);
// Row i of the source adjacency, decoded from its segment's start (references
// never leave a segment): the reference's reconstruct_row
// (ref_matrix.hpp:71-73).  std::out_of_range if i >= n.
std::vector<uint32_t> bv_reconstruct_row(const BvStream& s, uint32_t i);
HostCsr transpose_csr(const HostCsr& g);

// ---- biclique covers (biclique.cpp; reference include/cmv/biclique.hpp) ----
struct Biclique {                  // complete directed bipartite edge set sources x targets
  std::vector<uint32_t> sources;   // strictly ascending
  std::vector<uint32_t> targets;   // strictly ascending
};
struct BicliqueCover {             // edge-disjoint bicliques + residual edges, union = E
  uint32_t n = 0;
  std::vector<Biclique> bicliques;                    // emission order
  std::vector<std::pair<uint32_t, uint32_t>> residual;  // sorted (u, v)
  uint64_t compressed_size() const;                   // sum |S|+|C| + |residual| (biclique.hpp:33-34)
};
// Device operands of the product y = M [x ; T x] (csrc/bicover.cu).
struct CoverLayout {
  uint32_t n = 0;
  uint64_t nb = 0;
  std::vector<uint64_t> t_off, m_off;  // nb + 1, n + 1
  std::vector<uint32_t> t_cols, m_cols;
};
BicliqueCover extract_greedy(const HostCsr& g, uint64_t min_gain, uint64_t max_rounds, uint32_t per_round);
void validate_cover_structure(const BicliqueCover& c);
bool verify_cover(const BicliqueCover& c, const HostCsr& g);
std::string save_cover_text(const BicliqueCover& c);
BicliqueCover load_cover_text(const std::string& text);
void save_cover_file(const BicliqueCover& c, const std::string& path);
BicliqueCover load_cover_file(const std::string& path);
void build_cover_layout(const BicliqueCover& c, CoverLayout& L);

// ---- CBV1 container (bv_io.cpp): the BV stream on disk ----------------------
// The reference's container error types (rmv_io.hpp:13-22).
struct FormatError : std::runtime_error {  // unrecognised container: bad magic or version
  using std::runtime_error::runtime_error;
};
struct CorruptionError : std::runtime_error {  // recognised container, inconsistent contents
  using std::runtime_error::runtime_error;
};
std::vector<uint8_t> encode_bv_container(const BvStream& s);
BvStream decode_bv_container(const uint8_t* p, size_t len);
void save_bv_container(const BvStream& s, const std::string& path);
BvStream load_bv_container(const std::string& path);

}  // namespace cmvg
