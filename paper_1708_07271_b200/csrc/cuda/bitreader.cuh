// Device bit reader for MSB-first u32-word streams (layout documented in
// host/bits.hpp).  A 64-bit window `cur` holds `nb` valid bits (MSB-aligned);
// it is refilled one 32-bit word at a time so that nb >= 32 after every
// consume, which covers every code the layouts use (unary prefix <= 31 zeros,
// payload <= 32 bits).
#pragma once
#include <cstdint>

namespace cmvg {

struct DevBits {
  uint64_t cur;
  int nb;
  const uint32_t* p;

  __device__ __forceinline__ void init(const uint32_t* base, uint32_t byte_idx) {
    p = base + (byte_idx >> 2);
    int skip = (int)(byte_idx & 3) * 8;
    cur = ((uint64_t)p[0] << 32) | p[1];
    p += 2;
    cur <<= skip;
    nb = 64 - skip;
  }
  __device__ __forceinline__ void init_bit(const uint32_t* base, uint64_t bitpos) {
    p = base + (bitpos >> 5);
    int skip = (int)(bitpos & 31);
    cur = ((uint64_t)p[0] << 32) | p[1];
    p += 2;
    cur <<= skip;
    nb = 64 - skip;
    fill();
  }
  // absolute bit position of the next unread bit (stream base `base`)
  __device__ __forceinline__ uint64_t bitpos(const uint32_t* base) const {
    return ((uint64_t)(p - base) << 5) - (uint64_t)nb;
  }
  __device__ __forceinline__ void fill() {
    if (nb <= 32) {
      cur |= (uint64_t)(*p++) << (32 - nb);
      nb += 32;
    }
  }
  __device__ __forceinline__ void skip(int k) {
    cur <<= k;
    nb -= k;
    fill();
  }
  __device__ __forceinline__ uint32_t bits(int k) {  // 1 <= k <= 32
    uint32_t v = (uint32_t)(cur >> (64 - k));
    skip(k);
    return v;
  }
  __device__ __forceinline__ uint32_t unary() {
    int lz = __clzll(cur);
    skip(lz + 1);
    return (uint32_t)lz;
  }
  __device__ __forceinline__ uint32_t gamma() {
    int L = __clzll(cur);
    // unary(L) + L payload bits; consume the prefix then the payload
    skip(L + 1);
    uint32_t low = L ? (uint32_t)(cur >> (64 - L)) : 0u;
    if (L) skip(L);
    return ((1u << L) | low) - 1u;
  }
  // Z code of the device layout (host/bits.hpp zfix): h zeros, a one, then
  // v = x + 1 in 3h+3 bits.  Fast path when the whole code is in the window.
  __device__ __forceinline__ uint32_t zfix() {
    int h = __clzll(cur);
    int tot = 4 * h + 4;
    if (tot <= nb) {
      uint32_t v = (uint32_t)(cur >> (64 - tot)) - (1u << (3 * h + 3));
      skip(tot);
      return v - 1u;
    }
    skip(h + 1);
    int w = 3 * h + 3;
    uint32_t v = (uint32_t)(cur >> (64 - w));
    skip(w);
    return v - 1u;
  }
  template <int K>
  __device__ __forceinline__ uint32_t zeta() {
    int h = __clzll(cur);
    skip(h + 1);
    int s = (h + 1) * K;
    uint32_t t = 1u << (h * K);
    uint32_t u = (uint32_t)(cur >> (64 - (s - 1)));
    uint32_t r;
    if (u < t) {
      r = u;
      skip(s - 1);
    } else {
      r = (uint32_t)(cur >> (64 - s)) - t;
      skip(s);
    }
    return r + t - 1u;
  }
};

__device__ __forceinline__ int32_t unfold_i32(uint32_t u) {
  return (u & 1u) ? -(int32_t)((u + 1u) >> 1) : (int32_t)(u >> 1);
}

// Position-based reader used by the serial BV->CSR decoder: every get()
// re-reads from memory, so several independent cursors can walk the same
// stream.
struct PosBits {
  const uint32_t* w;
  uint64_t pos;
  __device__ __forceinline__ uint64_t peek64() const {
    uint64_t wi = pos >> 5;
    int off = (int)(pos & 31);
    uint64_t hi = ((uint64_t)w[wi] << 32) | w[wi + 1];
    uint64_t lo = w[wi + 2];
    return off ? (hi << off) | (lo >> (32 - off)) : hi;
  }
  __device__ __forceinline__ uint32_t bits(int k) {  // 1..32
    uint32_t v = (uint32_t)(peek64() >> (64 - k));
    pos += k;
    return v;
  }
  __device__ __forceinline__ uint32_t unary() {
    uint32_t total = 0;
    for (;;) {
      uint64_t v = peek64();
      if (v) {
        int lz = __clzll(v);
        pos += lz + 1;
        return total + lz;
      }
      pos += 64;
      total += 64;
    }
  }
  __device__ __forceinline__ uint64_t gamma() {
    uint32_t L = unary();
    uint64_t low = 0;
    if (L > 32) { low = (uint64_t)bits((int)L - 32) << 32; low |= bits(32); }
    else if (L) low = bits((int)L);
    return ((1ull << L) | low) - 1ull;
  }
  __device__ __forceinline__ uint64_t zeta(int k) {
    uint32_t h = unary();
    int s = (int)(h + 1) * k;
    uint64_t t = 1ull << (h * k);
    uint64_t u = bits(s - 1);
    uint64_t r;
    if (u < t) r = u;
    else r = ((u << 1) | bits(1)) - t;
    return r + t - 1ull;
  }
};

}  // namespace cmvg
