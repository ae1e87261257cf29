// Host-side bit I/O and the instantaneous codes used by the BV stream and the
// device (BV-D) layout.
//
// Bit order: a stream is a sequence of u32 words; stream bit p lives in word
// p/32 at bit (31 - p%32), i.e. MSB-first.  The device reader
// (cuda/bitreader.cuh) uses the same convention.
//
// Codes (all encode a natural number x >= 0 through v = x + 1 >= 1):
//   unary(x)  : x zero bits then a one bit.
//   gamma(x)  : L = floor(log2 v); unary(L) then the low L bits of v.
//   zeta_k(x) : h = floor(floor(log2 v)/k); unary(h); then r = v - 2^(hk) in a
//               minimal binary code over [0, 2^((h+1)k) - 2^(hk)):
//               with s = (h+1)k and t = 2^(hk), r < t takes s-1 bits (r),
//               otherwise s bits (r + t).
// These are the Elias gamma and Boldi-Vigna zeta codes the WebGraph BV format
// uses (PAPER.md:139-154 names the framework; SURVEY.md Appendix B lists the
// fields).  The exact bit layout is ours: no reference test pins it
// (SURVEY.md §8c), so parity is pinned at the decoded-adjacency level.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace cmvg {

inline int ilog2_u64(uint64_t v) { return 63 - __builtin_clzll(v); }

inline uint64_t fold_signed(int64_t d) {  // 0,-1,1,-2,2 -> 0,1,2,3,4
  return d >= 0 ? (uint64_t)d << 1 : (((uint64_t)(-d)) << 1) - 1;
}
inline int64_t unfold_signed(uint64_t u) {
  return (u & 1) ? -(int64_t)((u + 1) >> 1) : (int64_t)(u >> 1);
}

inline int unary_len(uint64_t x) { return (int)x + 1; }
// Device-layout zeta_3 variant with a fixed-width payload: h zeros, a one,
// then v = x + 1 itself in 3h+3 bits (the minimal-binary refinement is dropped
// so the code length 4h+4 depends on h alone).
inline int zfix_len(uint64_t x) { return 4 * (ilog2_u64(x + 1) / 3) + 4; }
inline int gamma_len(uint64_t x) { return 2 * ilog2_u64(x + 1) + 1; }
inline int zeta_len(uint64_t x, int k) {
  uint64_t v = x + 1;
  int h = ilog2_u64(v) / k;
  int s = (h + 1) * k;
  uint64_t t = 1ull << (h * k);
  uint64_t r = v - t;
  return h + 1 + (r < t ? s - 1 : s);
}

class BitWriter {
 public:
  std::vector<uint32_t> words;
  uint64_t nbits = 0;

  void put(uint64_t v, int k) {  // low k bits of v, MSB first; k <= 64
    while (k > 0) {
      int room = 32 - (int)(nbits & 31);
      if (room == 32) words.push_back(0);
      int take = k < room ? k : room;
      uint32_t chunk = (uint32_t)((v >> (k - take)) & ((take == 32) ? 0xffffffffu : ((1u << take) - 1)));
      words.back() |= chunk << (room - take);
      nbits += take;
      k -= take;
    }
  }
  void unary(uint64_t x) {
    while (x >= 32) { put(0, 32); x -= 32; }
    put(1, (int)x + 1);
  }
  void gamma(uint64_t x) {
    uint64_t v = x + 1;
    int L = ilog2_u64(v);
    unary(L);
    if (L) put(v, L);
  }
  void zeta(uint64_t x, int k) {
    uint64_t v = x + 1;
    int h = ilog2_u64(v) / k;
    int s = (h + 1) * k;
    uint64_t t = 1ull << (h * k);
    uint64_t r = v - t;
    unary(h);
    if (r < t) put(r, s - 1);
    else put(r + t, s);
  }
  void zfix(uint64_t x) {
    uint64_t v = x + 1;
    int h = ilog2_u64(v) / 3;
    unary(h);
    put(v, 3 * h + 3);
  }
  void align(int bits) {  // pad with zeros to a multiple of `bits`
    while (nbits % bits) {
      uint64_t need = bits - nbits % bits;
      put(0, need > 32 ? 32 : (int)need);
    }
  }
  void append(const BitWriter& o) {
    uint64_t left = o.nbits;
    for (size_t w = 0; left > 0; ++w) {
      int k = left >= 32 ? 32 : (int)left;
      put(o.words[w] >> (32 - k), k);
      left -= k;
    }
  }
};

class BitReader {
 public:
  BitReader(const uint32_t* w, uint64_t nwords, uint64_t pos = 0) : w_(w), nw_(nwords), pos_(pos) {}
  uint64_t pos() const { return pos_; }
  void seek(uint64_t p) { pos_ = p; }
  uint64_t get(int k) {  // k <= 64
    uint64_t v = 0;
    while (k > 0) {
      uint64_t wi = pos_ >> 5;
      if (wi >= nw_) throw std::runtime_error("BV stream truncated");
      int off = (int)(pos_ & 31);
      int avail = 32 - off;
      int take = k < avail ? k : avail;
      uint32_t word = w_[wi];
      uint32_t chunk = (word << off) >> (32 - take);
      v = (take == 64 ? 0 : (v << take)) | chunk;
      pos_ += take;
      k -= take;
    }
    return v;
  }
  uint64_t unary() {
    uint64_t x = 0;
    while (get(1) == 0) {
      if (++x > 4096) throw std::runtime_error("BV stream corrupt: runaway unary code");
    }
    return x;
  }
  uint64_t gamma() {
    uint64_t L = unary();
    if (L > 63) throw std::runtime_error("BV stream corrupt: gamma too long");
    uint64_t low = L ? get((int)L) : 0;
    return ((1ull << L) | low) - 1;
  }
  uint64_t zfix() {
    uint64_t h = unary();
    if (h > 20) throw std::runtime_error("stream corrupt: zfix too long");
    return get((int)(3 * h + 3)) - 1;
  }
  uint64_t zeta(int k) {
    uint64_t h = unary();
    if ((h + 1) * k > 62) throw std::runtime_error("BV stream corrupt: zeta too long");
    int s = (int)(h + 1) * k;
    uint64_t t = 1ull << (h * k);
    uint64_t u = get(s - 1);
    uint64_t r;
    if (u < t) r = u;
    else r = ((u << 1) | get(1)) - t;
    return r + t - 1;
  }

 private:
  const uint32_t* w_;
  uint64_t nw_;
  uint64_t pos_;
};

}  // namespace cmvg
