// CPU Boldi-Vigna codec: CSR -> canonical BV stream (encoder) and back
// (decoder).  The encoder is the format-level replacement of the reference's
// `compress(g, W)` (include/cmv/ref_matrix.hpp:58-69): it picks, per row, the
// reference in the window that minimises the encoded length, ties to the
// nearest candidate (ref_matrix.hpp:63-64), and only references when strictly
// shorter than the self-coded row (keep-rule, ref_matrix.hpp:64-65,
// PAPER.md:211-212).  Unlike `compress` it bounds chains at R (max_ref) and
// never references across a segment boundary.
//
// Row layout:
//   gamma(outdegree d)
//   if d > 0:  unary(r), r in [0, w] (0 = no reference)
//   if r > 0:  gamma(b); b explicit copy-block lengths, alternating
//              copy/skip starting with copy: the first as gamma(len), the
//              rest as gamma(len-1); the remaining reference entries form an
//              implicit last block (copy when b is even, skip when odd).
//   if d - copied > 0 (the "extra" list):
//              gamma(#intervals); per interval gamma(left gap) and
//              gamma(len - Lmin) -- the first left extreme sign-folded
//              relative to i, later ones as left - prev_end - 1;
//              residuals (count implied): zeta_k of the first sign-folded
//              relative to i, then zeta_k(gap - 1).
#include <cstring>
#include <stdexcept>
#include <string>

#include "bits.hpp"
#include "host.hpp"

namespace cmvg {
namespace {

struct Scratch {
  std::vector<uint32_t> extra;
  std::vector<uint32_t> runs;
};

// Bits of the "extra" part (intervals + residuals) of row i.
uint64_t extra_cost(const std::vector<uint32_t>& ex, uint32_t i, const BvParams& p) {
  if (ex.empty()) return 0;
  uint64_t bits = 0, nint = 0;
  bool first_int = true, first_res = true;
  uint64_t prev_end = 0;
  uint32_t prev_res = 0;
  size_t k = 0, n = ex.size();
  while (k < n) {
    size_t e = k + 1;
    while (e < n && ex[e] == ex[e - 1] + 1) ++e;
    size_t len = e - k;
    if (len >= p.min_interval) {
      ++nint;
      uint64_t left = ex[k];
      bits += first_int ? gamma_len(fold_signed((int64_t)left - (int64_t)i)) : gamma_len(left - prev_end - 1);
      bits += gamma_len(len - p.min_interval);
      first_int = false;
      prev_end = left + len;
    } else {
      for (size_t t = k; t < e; ++t) {
        bits += first_res ? zeta_len(fold_signed((int64_t)ex[t] - (int64_t)i), p.zeta_k)
                          : zeta_len(ex[t] - prev_res - 1, p.zeta_k);
        first_res = false;
        prev_res = ex[t];
      }
    }
    k = e;
  }
  return bits + gamma_len(nint);
}

void write_extra(BitWriter& bw, const std::vector<uint32_t>& ex, uint32_t i, const BvParams& p, BvStats& st) {
  if (ex.empty()) return;
  // two passes: intervals first, then residuals
  std::vector<std::pair<uint32_t, uint32_t>> ints;
  std::vector<uint32_t> res;
  size_t k = 0, n = ex.size();
  while (k < n) {
    size_t e = k + 1;
    while (e < n && ex[e] == ex[e - 1] + 1) ++e;
    if (e - k >= p.min_interval) ints.push_back({ex[k], (uint32_t)(e - k)});
    else
      for (size_t t = k; t < e; ++t) res.push_back(ex[t]);
    k = e;
  }
  bw.gamma(ints.size());
  uint64_t prev_end = 0;
  for (size_t t = 0; t < ints.size(); ++t) {
    uint64_t left = ints[t].first;
    if (t == 0) bw.gamma(fold_signed((int64_t)left - (int64_t)i));
    else bw.gamma(left - prev_end - 1);
    bw.gamma(ints[t].second - p.min_interval);
    prev_end = left + ints[t].second;
    st.interval_edges += ints[t].second;
  }
  st.intervals += ints.size();
  for (size_t t = 0; t < res.size(); ++t) {
    if (t == 0) bw.zeta(fold_signed((int64_t)res[t] - (int64_t)i), p.zeta_k);
    else bw.zeta(res[t] - res[t - 1] - 1, p.zeta_k);
  }
  st.residual_edges += res.size();
}

// Copy-block analysis of row L against reference list R: fills runs and the
// extra list; returns the number of copied entries.
uint32_t copy_blocks(const uint32_t* L, uint32_t dl, const uint32_t* R, uint32_t dr, Scratch& s) {
  s.extra.clear();
  s.runs.clear();
  uint32_t a = 0, copied = 0;
  bool cur_copy = true;
  uint32_t run = 0;
  for (uint32_t b = 0; b < dr; ++b) {
    uint32_t v = R[b];
    while (a < dl && L[a] < v) s.extra.push_back(L[a++]);
    bool in = (a < dl && L[a] == v);
    if (in) { ++a; ++copied; }
    if (in == cur_copy) ++run;
    else { s.runs.push_back(run); run = 1; cur_copy = in; }
  }
  s.runs.push_back(run);
  while (a < dl) s.extra.push_back(L[a++]);
  return copied;
}

uint64_t blocks_cost(const std::vector<uint32_t>& runs) {
  uint64_t b = runs.size() - 1;
  uint64_t bits = gamma_len(b);
  for (uint64_t k = 0; k < b; ++k) bits += k == 0 ? gamma_len(runs[k]) : gamma_len(runs[k] - 1);
  return bits;
}

}  // namespace

BvStream bv_encode(const HostCsr& g, const BvParams& p) {
  if (p.segment_rows == 0) throw std::invalid_argument("segment_rows must be >= 1");
  if (p.window > 255) throw std::invalid_argument("window must be <= 255");
  if (p.min_interval < 2) throw std::invalid_argument("min_interval must be >= 2");
  BvStream out;
  out.n = g.n;
  out.m = g.m();
  out.params = p;
  out.ref_dist.assign(g.n, 0);
  uint32_t seg = p.segment_rows;
  uint64_t nseg = ((uint64_t)g.n + seg - 1) / seg;
  std::vector<BitWriter> parts(nseg);
  std::vector<BvStats> pstats(nseg);
  const uint32_t R = p.max_ref ? p.max_ref : 0xffffffffu;
  parallel_for(nseg, [&](uint64_t sb, uint64_t se) {
    Scratch s, best;
    std::vector<uint32_t> depth(seg);
    for (uint64_t sg = sb; sg < se; ++sg) {
      uint32_t r0 = (uint32_t)(sg * seg), r1 = (uint32_t)std::min<uint64_t>(g.n, (sg + 1) * seg);
      BitWriter& bw = parts[sg];
      BvStats& st = pstats[sg];
      for (uint32_t i = r0; i < r1; ++i) {
        const uint32_t* L = g.row(i);
        uint32_t d = g.deg(i);
        bw.gamma(d);
        depth[i - r0] = 0;
        if (d == 0) continue;
        // self-coded candidate
        best.extra.assign(L, L + d);
        uint64_t best_bits = (p.window ? unary_len(0) : 0) + extra_cost(best.extra, i, p);
        uint32_t best_r = 0, best_copied = 0;
        for (uint32_t r = 1; r <= p.window && i >= r0 + r; ++r) {
          uint32_t j = i - r;
          if (depth[j - r0] >= R) continue;
          uint32_t dj = g.deg(j);
          if (dj == 0) continue;
          uint32_t copied = copy_blocks(L, d, g.row(j), dj, s);
          if (copied == 0) continue;
          uint64_t bits = unary_len(r) + blocks_cost(s.runs) + extra_cost(s.extra, i, p);
          if (bits < best_bits) {  // strict: ties keep the nearer candidate / the plain row
            best_bits = bits;
            best_r = r;
            best_copied = copied;
            std::swap(best.extra, s.extra);
            std::swap(best.runs, s.runs);
          }
        }
        if (p.window) bw.unary(best_r);
        if (best_r) {
          uint32_t b = (uint32_t)best.runs.size() - 1;
          bw.gamma(b);
          for (uint32_t k = 0; k < b; ++k) bw.gamma(k == 0 ? best.runs[k] : best.runs[k] - 1);
          depth[i - r0] = depth[i - best_r - r0] + 1;
          st.max_depth = std::max(st.max_depth, depth[i - r0]);
          st.rows_with_ref++;
          st.copied_edges += best_copied;
          st.minus_edges += g.deg(i - best_r) - best_copied;
          out.ref_dist[i] = (uint8_t)best_r;
        }
        write_extra(bw, best.extra, i, p, st);
      }
    }
  });
  out.segment_bit_offsets.assign(nseg + 1, 0);
  for (uint64_t s = 0; s < nseg; ++s) out.segment_bit_offsets[s + 1] = out.segment_bit_offsets[s] + parts[s].nbits;
  out.nbits = out.segment_bit_offsets[nseg];
  out.words.assign((out.nbits + 31) / 32 + 2, 0);  // +2 guard words for 64-bit peeks
  parallel_for(nseg, [&](uint64_t sb, uint64_t se) {
    for (uint64_t s = sb; s < se; ++s) {
      // splice segment s at an arbitrary bit offset; boundary words are shared
      // with neighbours, so write only whole interior words here and the
      // first/last partial words under a separate pass.
      uint64_t base = out.segment_bit_offsets[s];
      const BitWriter& bw = parts[s];
      uint64_t nb = bw.nbits;
      for (uint64_t q = 0; q < nb;) {
        uint64_t pos = base + q;
        int off = (int)(pos & 31);
        int take = (int)std::min<uint64_t>(32 - off, nb - q);
        // extract `take` bits of bw starting at q
        uint64_t wi = q >> 5;
        int qo = (int)(q & 31);
        uint64_t two = ((uint64_t)bw.words[wi] << 32) | (wi + 1 < bw.words.size() ? bw.words[wi + 1] : 0);
        uint32_t chunk = (uint32_t)((two << qo) >> (64 - take));
        uint32_t shifted = chunk << (32 - off - take);
        bool boundary = (off != 0) || (take != 32);
        if (boundary) __atomic_fetch_or(&out.words[pos >> 5], shifted, __ATOMIC_RELAXED);
        else out.words[pos >> 5] = shifted;
        q += take;
      }
    }
  });
  BvStats tot;
  for (auto& s : pstats) {
    tot.rows_with_ref += s.rows_with_ref;
    tot.copied_edges += s.copied_edges;
    tot.interval_edges += s.interval_edges;
    tot.intervals += s.intervals;
    tot.residual_edges += s.residual_edges;
    tot.minus_edges += s.minus_edges;
    tot.max_depth = std::max(tot.max_depth, s.max_depth);
  }
  tot.stream_bits = out.nbits;
  out.stats = tot;
  return out;
}

namespace {
// Decode rows [r0, rend) of segment sg (r0 = its first row) into c / roff
// (roff[k] = start of row r0 + k in c); ref_dist (optional) gets each row's
// reference distance.  The decoder validates every field and throws on a
// corrupt stream; full = rend is the segment end (then the segment's bit
// length is checked too).
struct SegScratch {
  std::vector<uint64_t> roff;
  std::vector<uint32_t> depth, copied, expanded, merged, tmp;
};
void decode_segment_rows(const BvStream& s, uint64_t sg, uint32_t rend, std::vector<uint32_t>& c, SegScratch& w,
                         uint8_t* ref_dist, uint32_t* degs) {
  const BvParams& p = s.params;
  const uint32_t seg = p.segment_rows;
  const uint32_t R = p.max_ref ? p.max_ref : 0xffffffffu;
  BitReader br(s.words.data(), s.words.size(), s.segment_bit_offsets[sg]);
  const uint32_t r0 = (uint32_t)(sg * seg), r1 = (uint32_t)std::min<uint64_t>(s.n, (sg + 1) * seg);
  std::vector<uint64_t>& roff = w.roff;
  std::vector<uint32_t>&depth = w.depth, &copied = w.copied, &expanded = w.expanded, &merged = w.merged, &tmp = w.tmp;
  depth.resize(seg);
  c.clear();
  roff.assign(1, 0);
  for (uint32_t i = r0; i < rend; ++i) {
    uint64_t d = br.gamma();
    depth[i - r0] = 0;
    if (d > s.n) throw std::runtime_error("BV stream corrupt: outdegree > n");
    if (d == 0) { roff.push_back(c.size()); if (degs) degs[i - r0] = 0; continue; }
    uint64_t r = p.window ? br.unary() : 0;
    if (r > p.window || (r && i < r0 + r)) throw std::runtime_error("BV stream corrupt: bad reference");
    copied.clear();
    if (r) {
      uint32_t j = i - (uint32_t)r;
      if (depth[j - r0] >= R) throw std::runtime_error("BV stream corrupt: chain exceeds R");
      depth[i - r0] = depth[j - r0] + 1;
      if (ref_dist) ref_dist[i] = (uint8_t)r;
      const uint32_t* Rl = c.data() + roff[j - r0];
      uint64_t dr = roff[j - r0 + 1] - roff[j - r0];
      uint64_t b = br.gamma();
      if (b > dr + 1) throw std::runtime_error("BV stream corrupt: too many copy blocks");
      uint64_t pos = 0;
      bool cp = true;
      for (uint64_t k = 0; k < b; ++k) {
        uint64_t len = k == 0 ? br.gamma() : br.gamma() + 1;
        if (pos + len > dr) throw std::runtime_error("BV stream corrupt: copy block overflow");
        if (cp) copied.insert(copied.end(), Rl + pos, Rl + pos + len);
        pos += len;
        cp = !cp;
      }
      if (cp) copied.insert(copied.end(), Rl + pos, Rl + dr);
    }
    if (copied.size() > d) throw std::runtime_error("BV stream corrupt: copied > outdegree");
    uint64_t extra = d - copied.size();
    expanded.clear();
    tmp.clear();
    if (extra) {
      uint64_t ni = br.gamma();
      uint64_t prev_end = 0, in_int = 0;
      for (uint64_t k = 0; k < ni; ++k) {
        int64_t left = k == 0 ? (int64_t)i + unfold_signed(br.gamma()) : (int64_t)(prev_end + br.gamma() + 1);
        uint64_t len = br.gamma() + p.min_interval;
        if (left < 0 || (uint64_t)left + len > s.n) throw std::runtime_error("BV stream corrupt: interval out of range");
        for (uint64_t t = 0; t < len; ++t) expanded.push_back((uint32_t)(left + t));
        prev_end = (uint64_t)left + len;
        in_int += len;
      }
      if (in_int > extra) throw std::runtime_error("BV stream corrupt: intervals exceed outdegree");
      uint64_t nres = extra - in_int;
      int64_t prev = 0;
      for (uint64_t k = 0; k < nres; ++k) {
        int64_t v = k == 0 ? (int64_t)i + unfold_signed(br.zeta(p.zeta_k)) : prev + (int64_t)br.zeta(p.zeta_k) + 1;
        if (v < 0 || v >= (int64_t)s.n) throw std::runtime_error("BV stream corrupt: residual out of range");
        tmp.push_back((uint32_t)v);
        prev = v;
      }
    }
    merged.resize(copied.size() + expanded.size());
    std::merge(copied.begin(), copied.end(), expanded.begin(), expanded.end(), merged.begin());
    size_t base = c.size();
    c.resize(base + merged.size() + tmp.size());
    std::merge(merged.begin(), merged.end(), tmp.begin(), tmp.end(), c.begin() + base);
    for (size_t t = base + 1; t < c.size(); ++t)
      if (c[t] <= c[t - 1]) throw std::runtime_error("BV stream corrupt: row not strictly increasing");
    roff.push_back(c.size());
    if (degs) degs[i - r0] = (uint32_t)d;
  }
  if (rend == r1 && br.pos() != s.segment_bit_offsets[sg + 1])
    throw std::runtime_error("BV stream corrupt: segment length mismatch");
}
}  // namespace

std::vector<uint32_t> bv_reconstruct_row(const BvStream& s, uint32_t i) {
  if (i >= s.n) throw std::out_of_range("reconstruct_row: row index out of range");
  const uint32_t seg = s.params.segment_rows;
  const uint64_t sg = i / seg;
  if (s.segment_bit_offsets.size() != ((uint64_t)s.n + seg - 1) / seg + 1)
    throw std::runtime_error("BV stream: bad segment table");
  std::vector<uint32_t> c;
  SegScratch w;
  decode_segment_rows(s, sg, i + 1, c, w, nullptr, nullptr);
  const uint32_t k = i - (uint32_t)(sg * seg);
  return std::vector<uint32_t>(c.begin() + w.roff[k], c.begin() + w.roff[k + 1]);
}

BvDecoded bv_decode(const BvStream& s) {
  const BvParams& p = s.params;
  uint32_t seg = p.segment_rows;
  uint64_t nseg = ((uint64_t)s.n + seg - 1) / seg;
  if (s.segment_bit_offsets.size() != nseg + 1) throw std::runtime_error("BV stream: bad segment table");
  std::vector<std::vector<uint32_t>> cols(nseg);
  std::vector<std::vector<uint32_t>> degs(nseg);
  BvDecoded out;
  out.ref_dist.assign(s.n, 0);
  parallel_for(nseg, [&](uint64_t sb, uint64_t se) {
    SegScratch w;
    for (uint64_t sg = sb; sg < se; ++sg) {
      const uint32_t r1 = (uint32_t)std::min<uint64_t>(s.n, (sg + 1) * seg);
      degs[sg].resize(r1 - sg * seg);
      decode_segment_rows(s, sg, r1, cols[sg], w, out.ref_dist.data(), degs[sg].data());
    }
  });
  HostCsr& g = out.csr;
  g.n = s.n;
  g.row_offsets.assign((size_t)s.n + 1, 0);
  std::vector<uint64_t> base(nseg + 1, 0);
  for (uint64_t k = 0; k < nseg; ++k) base[k + 1] = base[k] + cols[k].size();
  g.cols.resize(base[nseg]);
  parallel_for(nseg, [&](uint64_t sb, uint64_t se) {
    for (uint64_t k = sb; k < se; ++k) {
      uint64_t off = base[k];
      uint32_t r0 = (uint32_t)(k * seg);
      for (size_t t = 0; t < degs[k].size(); ++t) { off += degs[k][t]; g.row_offsets[r0 + t + 1] = off; }
      if (!cols[k].empty()) std::memcpy(g.cols.data() + base[k], cols[k].data(), cols[k].size() * 4);
      std::vector<uint32_t>().swap(cols[k]);
    }
  });
  return out;
}

HostCsr transpose_csr(const HostCsr& g) {
  HostCsr t;
  t.n = g.n;
  t.row_offsets.assign((size_t)g.n + 1, 0);
  for (uint32_t c : g.cols) t.row_offsets[c + 1]++;
  for (uint32_t v = 0; v < g.n; ++v) t.row_offsets[v + 1] += t.row_offsets[v];
  t.cols.resize(g.m());
  std::vector<uint64_t> cur(t.row_offsets.begin(), t.row_offsets.end() - 1);
  for (uint32_t u = 0; u < g.n; ++u)
    for (uint64_t e = g.row_offsets[u]; e < g.row_offsets[u + 1]; ++e) t.cols[cur[g.cols[e]]++] = u;
  return t;
}

}  // namespace cmvg
