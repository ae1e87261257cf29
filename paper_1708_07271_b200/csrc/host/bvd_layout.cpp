// Host builder of the BV-D device layout (see layout.hpp) from a decoded BV
// stream.  Preprocessing, run once per graph when a device handle is created.
#include "bvd_layout.hpp"

#include <cstring>
#include <stdexcept>

#include "bits.hpp"

namespace cmvg {
namespace {

struct RowParts {
  std::vector<uint32_t> minus, res;
  std::vector<std::pair<uint32_t, uint32_t>> ints;
};

// A' row of i against its BV reference i - r: minus = ref minus row, plus = row minus
// ref split into maximal runs >= Lmin (intervals) and the rest (residuals),
// which is exactly BV's extra-list split.
void split_row(const HostCsr& g, uint32_t i, uint32_t r, uint32_t lmin, RowParts& rp, std::vector<uint32_t>& plus) {
  rp.minus.clear();
  rp.res.clear();
  rp.ints.clear();
  plus.clear();
  const uint32_t* L = g.row(i);
  uint32_t dl = g.deg(i);
  if (r) {
    const uint32_t* R = g.row(i - r);
    uint32_t dr = g.deg(i - r);
    uint32_t a = 0, b = 0;
    while (a < dl || b < dr) {
      if (b >= dr || (a < dl && L[a] < R[b])) plus.push_back(L[a++]);
      else if (a >= dl || R[b] < L[a]) rp.minus.push_back(R[b++]);
      else { ++a; ++b; }
    }
  } else {
    plus.assign(L, L + dl);
  }
  size_t k = 0, n = plus.size();
  while (k < n) {
    size_t e = k + 1;
    while (e < n && plus[e] == plus[e - 1] + 1) ++e;
    if (e - k >= lmin) rp.ints.push_back({plus[k], (uint32_t)(e - k)});
    else
      for (size_t t = k; t < e; ++t) rp.res.push_back(plus[t]);
    k = e;
  }
}

inline uint32_t bits_of(uint64_t v) { return v ? 64u - (uint32_t)__builtin_clzll(v) : 0u; }

}  // namespace

BvdLayout build_bvd(const BvDecoded& dec, const BvParams& bp, const BvdOptions& opt) {
  const HostCsr& g = dec.csr;
  BvdLayout L;
  BvdDims& D = L.dims;
  const uint32_t B = opt.block_rows, W = opt.window;
  if (B == 0 || (B & (B - 1)) || B % bp.segment_rows || B > 4096)
    throw std::invalid_argument("block_rows must be a power of two <= 4096 and a multiple of the BV segment");
  if (W % 16 || W == 0) throw std::invalid_argument("window must be a positive multiple of 16");
  if (bp.window > 7) throw std::invalid_argument("the device layout supports BV windows w <= 7");
  D.n = g.n;
  D.block_rows = B;
  D.window = W;
  D.min_interval = bp.min_interval;
  D.nblocks = (uint32_t)(((uint64_t)g.n + B - 1) / B);
  D.max_depth = 0;
  const uint32_t nb = D.nblocks;
  std::vector<BitWriter> bstream(nb);
  L.blocks.resize(nb);
  std::vector<uint64_t> bbits(nb, 0), badds(nb, 0), bcodes(nb, 0), bgath(nb, 0), bin(nb, 0);
  std::vector<uint32_t> bdepth(nb, 0);
  parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
    std::vector<RowParts> rps(B);
    std::vector<uint32_t> plus, cols, depth(B), hdr(B), escs;
    BitWriter body;
    for (uint64_t b = b0; b < b1; ++b) {
      const uint32_t r0 = (uint32_t)(b * B), r1 = (uint32_t)std::min<uint64_t>(g.n, (b + 1) * B);
      const uint32_t nr = r1 - r0;
      cols.clear();
      escs.clear();
      body.words.clear();
      body.nbits = 0;
      uint64_t adds = 0, codes = 0;
      std::fill(hdr.begin(), hdr.end(), 0u);
      // pass 1: split rows, collect gathered columns, choose the x-window
      for (uint32_t k = 0; k < nr; ++k) {
        const uint32_t i = r0 + k;
        const uint32_t r = dec.ref_dist[i];
        if (r && k < r) throw std::runtime_error("BV-D: reference crosses a block");
        depth[k] = r ? depth[k - r] + 1 : 0;
        bdepth[b] = std::max(bdepth[b], depth[k]);
        RowParts& rp = rps[k];
        split_row(g, i, r, bp.min_interval, rp, plus);
        for (auto& iv : rp.ints) {
          cols.push_back(iv.first);
          cols.push_back(iv.first + iv.second - 1);
        }
        for (uint32_t c : rp.minus) cols.push_back(c);
        for (uint32_t c : rp.res) cols.push_back(c);
      }
      std::sort(cols.begin(), cols.end());
      uint64_t best = 0, best_lo = r0;
      for (size_t a = 0, e = 0; a < cols.size(); ++a) {
        while (e < cols.size() && cols[e] < (uint64_t)cols[a] + W) ++e;
        if (e - a > best) { best = e - a; best_lo = cols[a]; }
      }
      uint64_t lo = best_lo;
      if (!cols.empty()) {
        auto hi_it = std::lower_bound(cols.begin(), cols.end(), (uint32_t)std::min<uint64_t>(best_lo + W, 0xffffffffu));
        const uint32_t hi = *(hi_it - 1);
        const uint64_t slack = best_lo + W - 1 - hi;
        lo = best_lo >= slack / 2 ? best_lo - slack / 2 : 0;
      }
      lo &= ~15ull;
      auto inwin = [&](uint64_t c) { return c >= lo && c < lo + W; };
      uint64_t in_cnt = 0;
      for (uint32_t c : cols) in_cnt += inwin(c);
      bgath[b] = cols.size();
      bin[b] = in_cnt;
      // pass 2: headers (with the far flag) and bodies
      for (uint32_t k = 0; k < nr; ++k) {
        const uint32_t i = r0 + k;
        const uint32_t r = dec.ref_dist[i];
        const RowParts& rp = rps[k];
        const uint32_t nm = (uint32_t)rp.minus.size(), ns = (uint32_t)rp.res.size(), ni = (uint32_t)rp.ints.size();
        int64_t dmin = 0, dmax = 0;
        bool any = false, far = false;
        auto see = [&](uint32_t c) {
          const int64_t d = (int64_t)c - (int64_t)i;
          dmin = any ? std::min(dmin, d) : d;
          dmax = any ? std::max(dmax, d) : d;
          any = true;
          if (!inwin(c)) far = true;
        };
        for (uint32_t c : rp.minus) see(c);
        for (uint32_t c : rp.res) see(c);
        uint32_t wl = 0;
        for (auto& iv : rp.ints) {
          see(iv.first);
          if (!inwin((uint64_t)iv.first + iv.second - 1)) far = true;
          wl = std::max(wl, bits_of(iv.second - bp.min_interval));
        }
        // smallest wp with -2^(wp-1) <= d < 2^(wp-1) for every offset d
        uint32_t wp = 0;
        if (any)
          while (!(dmin >= -(int64_t)code_bias(wp) && dmax < (int64_t)(wp ? code_bias(wp) : 1))) ++wp;
        const int64_t bias = code_bias(wp);
        const bool esc = nm >= kHdrMinusEsc || ns >= kHdrResEsc || ni >= kHdrIntEsc;
        if (esc) {
          // all three counts escape together; the real counts go to the escape table
          hdr[k] = make_hdr(r, kHdrMinusEsc, kHdrResEsc, kHdrIntEsc, wp, wl, far);
          escs.push_back(k);
          escs.push_back(nm);
          escs.push_back(ns);
          escs.push_back(ni);
        } else {
          hdr[k] = make_hdr(r, nm, ns, ni, wp, wl, far);
        }
        for (uint32_t c : rp.minus) body.put((uint64_t)((int64_t)c - (int64_t)i + bias), (int)wp);
        for (uint32_t c : rp.res) body.put((uint64_t)((int64_t)c - (int64_t)i + bias), (int)wp);
        for (auto& iv : rp.ints) {
          body.put((uint64_t)((int64_t)iv.first - (int64_t)i + bias), (int)wp);
          body.put(iv.second - bp.min_interval, (int)wl);
        }
        codes += nm + ns + 2ull * ni;
        adds += (r ? 1 : 0) + nm + ns + 2ull * ni;
      }
      badds[b] = adds;
      bcodes[b] = codes;
      BitWriter& out = bstream[b];
      for (uint32_t q = 0; q < B; ++q) out.put(q < nr ? hdr[q] : 0u, 32);
      for (uint32_t e : escs) out.put(e, 32);
      bbits[b] = (uint64_t)nr * 32 + escs.size() * 32 + body.nbits;
      out.append(body);
      out.align(128);
      L.blocks[b].wlo = (uint32_t)lo;
      L.blocks[b].nwords = (uint32_t)(out.nbits / 32);
      L.blocks[b].nesc = (uint32_t)(escs.size() / 4);
    }
  });
  uint64_t off = 0, maxw = 0, g_all = 0, g_in = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    L.blocks[b].word_offset = off;
    off += L.blocks[b].nwords;
    maxw = std::max<uint64_t>(maxw, L.blocks[b].nwords);
    L.stats.row_bits += bbits[b];
    L.stats.codes += bcodes[b];
    L.adds_per_product += badds[b];
    g_all += bgath[b];
    g_in += bin[b];
    D.max_depth = std::max(D.max_depth, bdepth[b]);
  }
  D.max_block_words = (uint32_t)maxw;
  {
    std::vector<uint32_t> sz(nb);
    for (uint32_t b = 0; b < nb; ++b) sz[b] = L.blocks[b].nwords;
    std::sort(sz.begin(), sz.end());
    L.stats.p995_block_words = nb ? sz[std::min<uint64_t>(nb - 1, (uint64_t)(nb * 0.995))] : 0;
  }
  L.stats.window_coverage = g_all ? (double)g_in / (double)g_all : 1.0;
  L.words.assign(off + 8, 0);  // guard words
  parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
    for (uint64_t b = b0; b < b1; ++b)
      if (L.blocks[b].nwords)
        std::memcpy(L.words.data() + L.blocks[b].word_offset, bstream[b].words.data(), (size_t)L.blocks[b].nwords * 4);
  });
  L.stats.stream_bytes = off * 4;
  L.stats.block_table_bytes = (uint64_t)nb * sizeof(BvdBlockInfo);
  return L;
}

}  // namespace cmvg
