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

void write_gapped_zeta(BitWriter& bw, const std::vector<uint32_t>& v, uint32_t i, uint32_t k) {
  for (size_t t = 0; t < v.size(); ++t) {
    if (t == 0) bw.zeta(fold_signed((int64_t)v[0] - (int64_t)i), k);
    else bw.zeta(v[t] - v[t - 1] - 1, k);
  }
}

}  // namespace

BvdLayout build_bvd(const BvDecoded& dec, const BvParams& bp, const BvdOptions& opt) {
  const HostCsr& g = dec.csr;
  BvdLayout L;
  BvdDims& D = L.dims;
  uint32_t B = opt.block_rows, T = opt.lanes, W = opt.window;
  if (B == 0 || (B & (B - 1)) || B % bp.segment_rows) throw std::invalid_argument("block_rows must be a power of two and a multiple of the BV segment");
  if (T == 0 || T % 32 || T > 1024) throw std::invalid_argument("lanes must be a multiple of 32, <= 1024");
  if (W % 16 || W == 0) throw std::invalid_argument("window must be a positive multiple of 16");
  D.n = g.n;
  D.block_rows = B;
  D.lanes = T;
  D.row_bits = 0;
  while ((1u << D.row_bits) <= B) ++D.row_bits;  // field holds 0..B inclusive
  D.window = W;
  D.ref_bits = 0;
  while ((1u << D.ref_bits) <= bp.window) ++D.ref_bits;
  D.min_interval = bp.min_interval;
  D.zeta_k = bp.zeta_k;
  D.nblocks = (uint32_t)(((uint64_t)g.n + B - 1) / B);
  D.max_depth = 0;
  const uint32_t nb = D.nblocks;
  std::vector<BitWriter> bstream(nb);
  L.blocks.resize(nb);
  L.lanes.resize((uint64_t)nb * T);
  std::vector<uint64_t> bbits(nb, 0), badds(nb, 0);
  std::vector<uint32_t> bdepth(nb, 0);
  const uint32_t max_off = 1u << (32 - D.row_bits);
  parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
    RowParts rp;
    std::vector<uint32_t> plus, cols, depth(B);
    std::vector<BitWriter> rows(B);
    std::vector<uint64_t> cost(B + 1);
    for (uint64_t b = b0; b < b1; ++b) {
      uint32_t r0 = (uint32_t)(b * B), r1 = (uint32_t)std::min<uint64_t>(g.n, (b + 1) * B);
      uint32_t nr = r1 - r0;
      cols.clear();
      cost[0] = 0;
      uint64_t adds = 0;
      for (uint32_t k = 0; k < nr; ++k) {
        uint32_t i = r0 + k;
        uint32_t r = dec.ref_dist[i];
        if (r && k < r) throw std::runtime_error("BV-D: reference crosses a block");
        depth[k] = r ? depth[k - r] + 1 : 0;
        bdepth[b] = std::max(bdepth[b], depth[k]);
        split_row(g, i, r, bp.min_interval, rp, plus);
        BitWriter& bw = rows[k];
        bw.words.clear();
        bw.nbits = 0;
        bw.put(r, D.ref_bits);
        if (r) {
          bw.gamma(rp.minus.size());
          write_gapped_zeta(bw, rp.minus, i, bp.zeta_k);
        }
        bw.gamma(rp.ints.size());
        uint64_t prev_end = 0;
        for (size_t t = 0; t < rp.ints.size(); ++t) {
          uint64_t left = rp.ints[t].first;
          if (t == 0) bw.gamma(fold_signed((int64_t)left - (int64_t)i));
          else bw.gamma(left - prev_end - 1);
          bw.gamma(rp.ints[t].second - bp.min_interval);
          prev_end = left + rp.ints[t].second;
          cols.push_back((uint32_t)left);
          cols.push_back((uint32_t)(left + rp.ints[t].second - 1));
        }
        bw.gamma(rp.res.size());
        write_gapped_zeta(bw, rp.res, i, bp.zeta_k);
        for (uint32_t c : rp.minus) cols.push_back(c);
        for (uint32_t c : rp.res) cols.push_back(c);
        uint64_t ncodes = rp.minus.size() + rp.res.size();
        cost[k + 1] = cost[k] + 24 + 10 * ncodes + 14 * rp.ints.size();
        adds += (r ? 1 : 0) + rp.minus.size() + rp.res.size() + 2 * rp.ints.size();
        bbits[b] += bw.nbits;
      }
      badds[b] = adds;
      // contiguous, cost-balanced row ranges per lane
      std::vector<uint32_t> start(T + 1, nr);
      start[0] = 0;
      uint32_t k = 0;
      for (uint32_t t = 1; t < T; ++t) {
        uint64_t target = cost[nr] * t / T;
        while (k < nr && cost[k] < target) ++k;
        // pick the nearer of k-1 / k
        uint32_t cut = k;
        if (k > start[t - 1] && k > 0 && target - cost[k - 1] < cost[k] - target) cut = k - 1;
        if (cut < start[t - 1]) cut = start[t - 1];
        start[t] = cut;
      }
      start[T] = nr;
      BitWriter& out = bstream[b];
      for (uint32_t t = 0; t < T; ++t) {
        out.align(8);
        uint64_t byte = out.nbits / 8;
        if (byte >= max_off) throw std::runtime_error("BV-D: block stream too large for the lane table");
        L.lanes[b * T + t] = (uint32_t)(byte << D.row_bits) | start[t];
        for (uint32_t q = start[t]; q < start[t + 1]; ++q) out.append(rows[q]);
      }
      out.align(128);
      // x window: the W-range covering the most gathered columns
      std::sort(cols.begin(), cols.end());
      uint32_t best = 0, best_lo = r0;
      for (size_t a = 0, e = 0; a < cols.size(); ++a) {
        while (e < cols.size() && cols[e] < (uint64_t)cols[a] + W) ++e;
        if (e - a > best) { best = (uint32_t)(e - a); best_lo = cols[a]; }
      }
      // centre the covering range inside the window, align to 16
      uint64_t lo = best_lo;
      if (!cols.empty()) {
        auto hi_it = std::lower_bound(cols.begin(), cols.end(), (uint64_t)best_lo + W);
        uint32_t hi = *(hi_it - 1);
        uint64_t slack = (uint64_t)best_lo + W - 1 - hi;
        lo = best_lo >= slack / 2 ? best_lo - slack / 2 : 0;
      }
      lo &= ~15ull;
      L.blocks[b].wlo = (uint32_t)lo;
      L.blocks[b].nwords = (uint32_t)(out.nbits / 32);
    }
  });
  uint64_t off = 0, maxw = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    L.blocks[b].word_offset = off;
    off += L.blocks[b].nwords;
    maxw = std::max<uint64_t>(maxw, L.blocks[b].nwords);
    L.stats.row_bits += bbits[b];
    L.adds_per_product += badds[b];
    D.max_depth = std::max(D.max_depth, bdepth[b]);
  }
  D.max_block_words = (uint32_t)maxw;
  L.words.assign(off + 8, 0);  // guard words
  parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
    for (uint64_t b = b0; b < b1; ++b)
      if (L.blocks[b].nwords)
        std::memcpy(L.words.data() + L.blocks[b].word_offset, bstream[b].words.data(), (size_t)L.blocks[b].nwords * 4);
  });
  L.stats.stream_bytes = off * 4;
  L.stats.lane_table_bytes = (uint64_t)nb * T * 4;
  L.stats.block_table_bytes = (uint64_t)nb * sizeof(BvdBlockInfo);
  return L;
}

}  // namespace cmvg
