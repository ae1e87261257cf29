// CBV1: the on-disk container of a canonical BV stream,
// modelled on the reference's RMV1 container for ReferencedMatrix
// (rmv_io.hpp:31-49): a magic and a version byte, fixed-width
// little-endian header fields, the body, and strict validation on load --
// FormatError for an unrecognised container (bad magic or version),
// CorruptionError for a recognised one with inconsistent contents
// (truncation, trailing bytes, checksum, invariant violations, a stream that
// does not decode to m edges).  No partial results.  Encoding is
// deterministic: equal streams give identical bytes.
//
// Layout (little-endian):
//   "CBV1" | u8 version = 1 | 3 zero bytes
//   u32 n | u64 m | u32 window, max_ref, min_interval, zeta_k, segment_rows | u32 0
//   u64 nbits | u64 nseg | u64 segment_bit_offsets[nseg + 1]
//   u32 words[ceil(nbits / 32)]        (MSB-first bit stream, host/bits.hpp)
//   u64 FNV-1a of every preceding byte
#include <mutex>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>

#include "host.hpp"

namespace cmvg {

namespace {
constexpr char kMagic[4] = {'C', 'B', 'V', '1'};
constexpr uint8_t kVersion = 1;
constexpr size_t kHeadBytes = 8 + 4 + 8 + 6 * 4 + 8 + 8;

uint64_t fnv1a(const uint8_t* p, size_t len) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
template <typename T>
void put(std::vector<uint8_t>& o, T v) {
  uint8_t b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));  // host is little-endian (x86-64)
  o.insert(o.end(), b, b + sizeof(T));
}
template <typename T>
T get(const uint8_t* p, size_t& pos) {
  T v;
  std::memcpy(&v, p + pos, sizeof(T));
  pos += sizeof(T);
  return v;
}
}  // namespace

std::vector<uint8_t> encode_bv_container(const BvStream& s) {
  const uint64_t nw = (s.nbits + 31) / 32;
  const uint64_t nseg = s.segment_bit_offsets.empty() ? 0 : s.segment_bit_offsets.size() - 1;
  if (s.words.size() < nw) throw std::invalid_argument("BV stream: fewer words than bits");
  std::vector<uint8_t> o;
  o.reserve(kHeadBytes + 8 * (nseg + 1) + 4 * nw + 8);
  o.insert(o.end(), kMagic, kMagic + 4);
  put<uint8_t>(o, kVersion);
  put<uint8_t>(o, 0);
  put<uint16_t>(o, 0);
  put<uint32_t>(o, s.n);
  put<uint64_t>(o, s.m);
  put<uint32_t>(o, s.params.window);
  put<uint32_t>(o, s.params.max_ref);
  put<uint32_t>(o, s.params.min_interval);
  put<uint32_t>(o, s.params.zeta_k);
  put<uint32_t>(o, s.params.segment_rows);
  put<uint32_t>(o, 0);
  put<uint64_t>(o, s.nbits);
  put<uint64_t>(o, nseg);
  for (uint64_t v : s.segment_bit_offsets) put<uint64_t>(o, v);
  for (uint64_t i = 0; i < nw; ++i) put<uint32_t>(o, s.words[i]);
  put<uint64_t>(o, fnv1a(o.data(), o.size()));
  return o;
}

BvStream decode_bv_container(const uint8_t* p, size_t len) {
  if (len < 5 || std::memcmp(p, kMagic, 4) != 0) throw FormatError("CBV1: bad magic");
  if (p[4] != kVersion) throw FormatError("CBV1: unsupported version " + std::to_string(p[4]));
  if (len < kHeadBytes) throw CorruptionError("CBV1: truncated header");
  size_t pos = 5;
  if (get<uint8_t>(p, pos) != 0 || get<uint16_t>(p, pos) != 0) throw CorruptionError("CBV1: corrupt header padding");
  BvStream s;
  s.n = get<uint32_t>(p, pos);
  s.m = get<uint64_t>(p, pos);
  s.params.window = get<uint32_t>(p, pos);
  s.params.max_ref = get<uint32_t>(p, pos);
  s.params.min_interval = get<uint32_t>(p, pos);
  s.params.zeta_k = get<uint32_t>(p, pos);
  s.params.segment_rows = get<uint32_t>(p, pos);
  if (get<uint32_t>(p, pos) != 0) throw CorruptionError("CBV1: corrupt header padding");
  s.nbits = get<uint64_t>(p, pos);
  const uint64_t nseg = get<uint64_t>(p, pos);
  // sizes before any allocation (a corrupt header must not allocate terabytes)
  const uint64_t nw = (s.nbits + 31) / 32;
  if (s.nbits > (uint64_t)len * 8 || nseg > len / 8) throw CorruptionError("CBV1: truncated body");
  const uint64_t want = kHeadBytes + 8 * (nseg + 1) + 4 * nw + 8;
  if (len < want) throw CorruptionError("CBV1: truncated body");
  if (len > want) throw CorruptionError("CBV1: trailing bytes");
  {
    size_t cpos = len - 8;
    if (fnv1a(p, len - 8) != get<uint64_t>(p, cpos)) throw CorruptionError("CBV1: checksum mismatch (corrupt)");
  }
  const BvParams& q = s.params;
  if (q.window < 1 || q.window > 255 || q.min_interval < 2 || q.zeta_k < 1 || q.zeta_k > 16 || q.segment_rows == 0)
    throw CorruptionError("CBV1: corrupt parameters");
  if (nseg != ((uint64_t)s.n + q.segment_rows - 1) / q.segment_rows) throw CorruptionError("CBV1: corrupt segment count");
  s.segment_bit_offsets.resize(nseg + 1);
  for (auto& v : s.segment_bit_offsets) v = get<uint64_t>(p, pos);
  if (s.segment_bit_offsets.front() != 0 || s.segment_bit_offsets.back() != s.nbits)
    throw CorruptionError("CBV1: corrupt segment table");
  for (uint64_t i = 0; i < nseg; ++i)
    if (s.segment_bit_offsets[i] > s.segment_bit_offsets[i + 1]) throw CorruptionError("CBV1: corrupt segment table");
  s.words.resize(nw + 2, 0u);  // two zero guard words, as the encoder leaves them
  for (uint64_t i = 0; i < nw; ++i) s.words[i] = get<uint32_t>(p, pos);
  // every structural invariant: the stream decodes (the decoder validates
  // every field) to exactly m edges with references inside the window
  BvDecoded d;
  try {
    d = bv_decode(s);
  } catch (const std::exception& e) {
    throw CorruptionError(std::string("CBV1: stream does not decode (corrupt): ") + e.what());
  }
  if (d.csr.m() != s.m) throw CorruptionError("CBV1: corrupt stream: edge count differs from the header");
  s.stats = BvStats{};
  s.stats.stream_bits = s.nbits;
  s.ref_dist = d.ref_dist;
  std::vector<uint32_t> depth(s.n, 0);
  for (uint32_t i = 0; i < s.n; ++i) {
    const uint32_t r = d.ref_dist[i];
    if (r) {
      ++s.stats.rows_with_ref;
      depth[i] = depth[i - r] + 1;
      s.stats.max_depth = std::max(s.stats.max_depth, depth[i]);
    }
  }
  // the encoder's edge statistics, recomputed from the decoded rows: copied =
  // row and reference in common, minus = the reference's other entries, the
  // extra entries split into maximal runs >= Lmin (intervals) and residuals
  const HostCsr& g = d.csr;
  std::mutex mu;
  parallel_for(s.n, [&](uint64_t b0, uint64_t b1) {
    BvStats t;
    for (uint64_t i = b0; i < b1; ++i) {
      const uint32_t r = d.ref_dist[i];
      const uint32_t* L = g.row((uint32_t)i);
      const uint32_t dl = g.deg((uint32_t)i);
      uint64_t common = 0;
      uint32_t run = 0, prev = 0;
      bool have = false;
      auto extra = [&](uint32_t c) {  // extras arrive in increasing order
        if (have && c == prev + 1) {
          ++run;
        } else {
          if (run) {
            if (run >= s.params.min_interval) {
              t.interval_edges += run;
              ++t.intervals;
            } else {
              t.residual_edges += run;
            }
          }
          run = 1;
        }
        prev = c;
        have = true;
      };
      if (r) {
        const uint32_t* R = g.row((uint32_t)i - r);
        const uint32_t dr = g.deg((uint32_t)i - r);
        uint32_t a = 0, b = 0;
        while (a < dl) {
          if (b < dr && R[b] < L[a]) ++b;
          else if (b < dr && R[b] == L[a]) { ++common; ++a; ++b; }
          else extra(L[a++]);
        }
        t.copied_edges += common;
        t.minus_edges += dr - common;
      } else {
        for (uint32_t a = 0; a < dl; ++a) extra(L[a]);
      }
      if (run) {
        if (run >= s.params.min_interval) {
          t.interval_edges += run;
          ++t.intervals;
        } else {
          t.residual_edges += run;
        }
      }
    }
    std::lock_guard<std::mutex> lk(mu);
    s.stats.copied_edges += t.copied_edges;
    s.stats.minus_edges += t.minus_edges;
    s.stats.interval_edges += t.interval_edges;
    s.stats.intervals += t.intervals;
    s.stats.residual_edges += t.residual_edges;
  });
  return s;
}

void save_bv_container(const BvStream& s, const std::string& path) {
  const std::vector<uint8_t> b = encode_bv_container(s);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw std::invalid_argument("CBV1: cannot open " + path + " for writing");
  f.write(reinterpret_cast<const char*>(b.data()), (std::streamsize)b.size());
  if (!f) throw std::runtime_error("CBV1: write failed: " + path);
}

BvStream load_bv_container(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::invalid_argument("CBV1: cannot open " + path);
  std::vector<uint8_t> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  return decode_bv_container(b.data(), b.size());
}

}  // namespace cmvg
