// Host builder of the BV-D device layout (see layout.hpp) from a decoded BV
// stream.  Preprocessing, run once per graph when a device handle is created.
#include "bvd_layout.hpp"

#include <cstring>
#include <stdexcept>

#include "bits.hpp"
#include "bvf_block.hpp"

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>

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

// LSD radix sort (two 16-bit digits): the per-block column lists (~10^4
// entries) sort ~5x faster than with std::sort
void radix_sort_u32(std::vector<uint32_t>& v) {
  if (v.size() < 256) {
    std::sort(v.begin(), v.end());
    return;
  }
  thread_local std::vector<uint32_t> tmp;
  thread_local std::vector<uint32_t> cnt;
  tmp.resize(v.size());
  for (int pass = 0; pass < 2; ++pass) {
    const int sh = 16 * pass;
    cnt.assign(65537, 0);
    for (uint32_t x : v) ++cnt[((x >> sh) & 0xffffu) + 1];
    for (size_t d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
    for (uint32_t x : v) tmp[cnt[(x >> sh) & 0xffffu]++] = x;
    v.swap(tmp);
  }
}

struct RowMeta {
  uint32_t r, nm, ns, ni, wp, wl;
  bool far;
  uint64_t bit0, nbits;  // the row's body within the block's BV-D body stream
};

// 32 bits of `w` starting at bit `pos`, bits at or past `end` zero (MSB first)
inline uint32_t bits32(const std::vector<uint32_t>& w, uint64_t pos, uint64_t end) {
  if (pos >= end) return 0u;
  const uint64_t wi = pos >> 5;
  const uint32_t sh = (uint32_t)(pos & 31);
  uint64_t win = (uint64_t)w[wi] << 32;
  if (wi + 1 < w.size()) win |= w[wi + 1];
  uint32_t v = (uint32_t)((win << sh) >> 32);
  const uint64_t left = end - pos;
  if (left < 32) v &= ~0u << (32 - left);
  return v;
}

// BV-S block stream from the block's rows (layout.hpp).  Units and their
// codes live in flat per-block arrays (no per-unit allocations).
struct Unit {
  uint32_t k, r, nm, np, ni;
  bool primary;
  uint32_t pc0, iw0, w0, nw;  // near: codes at pcs[pc0, +np), intervals at iws[iw0, +ni); else words at wds[w0, +nw)
};
struct URow {  // a row's units (adjacent lanes when there is more than one)
  uint32_t k, u0, nu;
  bool c32, far;
};

void emit_bvs(const RowParts* rps, const RowMeta* meta, const BitWriter& body, uint32_t nr, uint64_t wlo, uint32_t W,
              uint32_t lmin, std::vector<uint32_t>& so, BvsStats& st) {
  auto inwin = [&](uint64_t c) { return c >= wlo && c < wlo + W; };
  auto off_ok = [&](uint32_t c) {
    const int64_t d = (int64_t)c - (int64_t)wlo;
    return d >= -(int64_t)kBvsBias16 && d < (int64_t)kBvsBias16;
  };
  auto code16 = [&](uint32_t c) { return (uint32_t)((int64_t)c - (int64_t)wlo + kBvsBias16); };
  thread_local std::vector<Unit> units;
  thread_local std::vector<uint16_t> pcs;
  thread_local std::vector<uint32_t> iws, wds;
  thread_local std::vector<URow> single, multi;
  units.clear();
  pcs.clear();
  iws.clear();
  wds.clear();
  single.clear();
  multi.clear();
  std::vector<uint32_t> hrows;
  for (uint32_t k = 0; k < nr; ++k) {
    const RowParts& rp = rps[k];
    const uint32_t nm = (uint32_t)rp.minus.size(), np = nm + (uint32_t)rp.res.size(), ni = (uint32_t)rp.ints.size();
    const uint32_t nu = std::max<uint32_t>(
        1, std::max((np + kBvsUnitPts - 1) / kBvsUnitPts, (ni + kBvsUnitInts - 1) / kBvsUnitInts));
    if (nu > kBvsMaxUnits) {
      hrows.push_back(k);
      continue;
    }
    auto pt = [&](uint32_t t) { return t < nm ? rp.minus[t] : rp.res[t - nm]; };
    URow row{k, (uint32_t)units.size(), nu, false, false};
    for (uint32_t t = 0; t < np; ++t) {
      row.c32 |= !off_ok(pt(t));
      row.far |= !inwin(pt(t));
    }
    for (const auto& iv : rp.ints) {
      row.c32 |= !off_ok(iv.first) || (iv.second - lmin) >= 65536u;
      row.far |= !inwin(iv.first) || !inwin((uint64_t)iv.first + iv.second - 1);
    }
    for (uint32_t j = 0; j < nu; ++j) {
      Unit u{};
      u.k = k;
      u.primary = j == 0;
      u.r = meta[k].r;
      // balanced split: unit j takes points [j np / nu, (j+1) np / nu), same for intervals
      const uint32_t p0 = (uint32_t)((uint64_t)j * np / nu), p1 = (uint32_t)((uint64_t)(j + 1) * np / nu);
      const uint32_t q0 = (uint32_t)((uint64_t)j * ni / nu), q1 = (uint32_t)((uint64_t)(j + 1) * ni / nu);
      u.np = p1 - p0;
      u.ni = q1 - q0;
      u.nm = nm > p0 ? std::min(nm, p1) - p0 : 0;
      u.pc0 = (uint32_t)pcs.size();
      u.iw0 = (uint32_t)iws.size();
      u.w0 = (uint32_t)wds.size();
      if (!row.c32 && !row.far) {
        for (uint32_t t = p0; t < p1; ++t)
          pcs.push_back((uint16_t)(bvs_pad_index((uint32_t)(pt(t) - wlo)) | (t < nm ? 0x8000u : 0u)));
        for (uint32_t t = q0; t < q1; ++t) iws.push_back(((uint32_t)(rp.ints[t].first - wlo) << 16) | rp.ints[t].second);
      } else if (!row.c32) {
        for (uint32_t t = p0; t < p1; t += 2) {
          const uint32_t hi = code16(pt(t)), lo = t + 1 < p1 ? code16(pt(t + 1)) : 0u;
          wds.push_back((hi << 16) | lo);
        }
        for (uint32_t t = q0; t < q1; ++t) wds.push_back((code16(rp.ints[t].first) << 16) | (rp.ints[t].second - lmin));
      } else {
        for (uint32_t t = p0; t < p1; ++t) wds.push_back(pt(t));
        for (uint32_t t = q0; t < q1; ++t) {
          wds.push_back(rp.ints[t].first);
          wds.push_back(rp.ints[t].second - lmin);
        }
      }
      u.nw = (uint32_t)wds.size() - u.w0;
      units.push_back(u);
    }
    (nu == 1 ? single : multi).push_back(row);
  }
  // slices: lists of unit lanes; groups (class32, far) never share a slice
  struct Slice {
    std::vector<uint32_t> lanes;  // unit indices
    bool c32, far, multi;
    uint32_t maxnu = 1;           // most units of one row in the slice
  };
  std::vector<Slice> slices;
  auto gid = [](const URow& r) { return (r.c32 ? 0 : 2) + (r.far ? 0 : 1); };
  // multi-unit rows: by per-unit load (so a slice's lanes have similar work),
  // then unit count, packed first-fit
  auto load = [&](const URow& r) {
    uint32_t p = 0, i = 0;
    for (uint32_t q = 0; q < r.nu; ++q) {
      p = std::max(p, units[r.u0 + q].np);
      i = std::max(i, units[r.u0 + q].ni);
    }
    return p + 2 * i;
  };
  std::stable_sort(multi.begin(), multi.end(), [&](const URow& a, const URow& b) {
    if (gid(a) != gid(b)) return gid(a) < gid(b);
    if (load(a) != load(b)) return load(a) > load(b);
    return a.nu > b.nu;
  });
  for (size_t a = 0; a < multi.size();) {
    size_t e = a;
    while (e < multi.size() && gid(multi[e]) == gid(multi[a])) ++e;
    const size_t first = slices.size();
    for (size_t q = a; q < e; ++q) {
      const URow& row = multi[q];
      size_t t = first;
      while (t < slices.size() && slices[t].lanes.size() + row.nu > 32) ++t;
      if (t == slices.size()) slices.push_back(Slice{{}, row.c32, row.far, true});
      for (uint32_t u = 0; u < row.nu; ++u) slices[t].lanes.push_back(row.u0 + u);
      slices[t].maxnu = std::max(slices[t].maxnu, row.nu);
    }
    a = e;
  }
  // single-unit rows: by (#intervals, #points) desc, dealt 32 per slice
  std::stable_sort(single.begin(), single.end(), [&](const URow& a, const URow& b) {
    if (gid(a) != gid(b)) return gid(a) < gid(b);
    const Unit &ua = units[a.u0], &ub = units[b.u0];
    if (ua.ni != ub.ni) return ua.ni > ub.ni;
    return ua.np > ub.np;
  });
  for (size_t a = 0; a < single.size();) {
    Slice sl{{}, single[a].c32, single[a].far, false};
    size_t e = a;
    while (e < single.size() && e - a < 32 && gid(single[e]) == gid(single[a])) sl.lanes.push_back(single[e++].u0);
    slices.push_back(std::move(sl));
    a = e;
  }
  const uint32_t nsl = (uint32_t)slices.size(), nh = (uint32_t)hrows.size();
  if (nsl > 0xffffu || nh > 0xffffu) throw std::runtime_error("BV-S: block too large");
  {
    // Static warp schedule: longest-processing-time assignment of the slices
    // to the kBvsWarps warps of a CTA by an instruction-count estimate, the
    // table reordered so warp w owns entries [start_w, start_{w+1}) -- no
    // ticket round trips, and the warps reach the chain barrier together.
    std::vector<uint32_t> cost(nsl), ord(nsl);
    for (uint32_t s = 0; s < nsl; ++s) {
      const Slice& sl = slices[s];
      uint32_t mnp = 0, mni = 0;
      for (uint32_t ui : sl.lanes) {
        mnp = std::max(mnp, units[ui].np);
        mni = std::max(mni, units[ui].ni);
      }
      uint32_t rounds = 0;
      while ((1u << rounds) < sl.maxnu) ++rounds;
      const bool nearc16 = !sl.c32 && !sl.far;
      cost[s] = 110u + (nearc16 ? 27u * ((mnp + 1) / 2) + 35u * mni : 22u * mnp + 60u * mni) + 30u * rounds;
      ord[s] = s;
    }
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return cost[a] > cost[b]; });
    std::vector<std::vector<uint32_t>> bins(kBvsWarps);
    std::vector<uint64_t> loadw(kBvsWarps, 0);
    for (uint32_t s : ord) {
      const uint32_t w = (uint32_t)(std::min_element(loadw.begin(), loadw.end()) - loadw.begin());
      bins[w].push_back(s);
      loadw[w] += cost[s];
    }
    std::vector<Slice> sorted;
    sorted.reserve(nsl);
    so.assign(kBvsHead + 2 * nsl, 0u);
    uint16_t* starts = reinterpret_cast<uint16_t*>(&so[kBvsWarpTab]);
    for (uint32_t w = 0; w < kBvsWarps; ++w) {
      starts[w] = (uint16_t)sorted.size();
      for (uint32_t s : bins[w]) sorted.push_back(std::move(slices[s]));
    }
    starts[kBvsWarps] = (uint16_t)sorted.size();
    slices.swap(sorted);
  }
  so[0] = nsl | (nh << 16);
  for (uint32_t s = 0; s < nsl; ++s) {
    const Slice& sl = slices[s];
    const bool nearc16 = !sl.c32 && !sl.far;
    so[kBvsHead + 2 * s] = (uint32_t)so.size();
    uint32_t mnp = 0, mni = 0, nq = 0;
    for (uint32_t ui : sl.lanes) {
      const Unit& u = units[ui];
      mnp = std::max(mnp, u.np);
      mni = std::max(mni, u.ni);
      nq = std::max<uint32_t>(nq, u.nw);
      st.lane_words_used += nearc16 ? (u.np + 1) / 2 + u.ni : u.nw;
      st.lane_iters_used += u.np + u.ni;
    }
    if (nearc16) nq = (mnp + 1) / 2 + mni;  // rectangular: points then intervals
    uint32_t rounds = 0;
    while ((1u << rounds) < sl.maxnu) ++rounds;
    so.push_back(make_smeta(mnp, mni, sl.c32, sl.far, sl.multi, rounds));
    so[kBvsHead + 2 * s + 1] = so.back();  // the table repeats the meta word
    for (size_t l = 0; l < 32; ++l) {
      if (l < sl.lanes.size()) {
        const Unit& u = units[sl.lanes[l]];
        so.push_back(make_uh(u.primary, u.primary ? u.k : 0u, u.primary ? u.r : 0u, u.nm, u.np, u.ni));
      } else {
        so.push_back(0u);
      }
    }
    const size_t b0 = so.size();
    so.resize(b0 + (size_t)nq * 32, 0u);
    if (nearc16) {
      // every lane: (mnp + 1) / 2 point words (pad codes read the window's
      // zero entry) then mni interval words (0 = empty interval)
      const uint32_t zc = bvs_pad_index(W), mnpw = (mnp + 1) / 2;
      for (size_t l = 0; l < 32; ++l) {
        const Unit* u = l < sl.lanes.size() ? &units[sl.lanes[l]] : nullptr;
        for (uint32_t q = 0; q < mnpw; ++q) {
          const uint32_t c0 = u && 2 * q < u->np ? pcs[u->pc0 + 2 * q] : zc;
          const uint32_t c1 = u && 2 * q + 1 < u->np ? pcs[u->pc0 + 2 * q + 1] : zc;
          so[b0 + (size_t)q * 32 + l] = (c0 << 16) | c1;
        }
        for (uint32_t q = 0; q < mni; ++q) so[b0 + (size_t)(mnpw + q) * 32 + l] = u && q < u->ni ? iws[u->iw0 + q] : 0u;
      }
    } else {
      for (size_t l = 0; l < sl.lanes.size(); ++l) {
        const Unit& u = units[sl.lanes[l]];
        for (uint32_t q = 0; q < u.nw; ++q) so[b0 + (size_t)q * 32 + l] = wds[u.w0 + q];
      }
    }
    st.lane_words += (uint64_t)nq * 32;
    st.lane_iters += 32ull * (mnp + mni);
  }
  so[1] = (uint32_t)so.size();
  BitWriter hs;
  uint32_t items = 0;
  for (uint32_t k : hrows) {
    const RowMeta& m = meta[k];
    so.push_back(make_sa(k, m.r, m.wp, m.wl, m.far));
    so.push_back(m.nm);
    so.push_back(m.ns);
    so.push_back(m.ni);
    so.push_back((uint32_t)hs.nbits);
    so.push_back(items);
    items += heavy_chunks(m.nm + m.ns);
    for (uint64_t p = m.bit0, e = m.bit0 + m.nbits; p < e; p += 32) {
      const uint32_t take = (uint32_t)std::min<uint64_t>(32, e - p);
      hs.put(bits32(body.words, p, e) >> (32 - take), (int)take);
    }
  }
  so[2] = (uint32_t)so.size();
  so.insert(so.end(), hs.words.begin(), hs.words.end());
  while (so.size() % 4) so.push_back(0u);
  st.slices += nsl;
  st.heavy_rows += nh;
  st.heavy_chunks += items;
}

// BV-T block stream (layout.hpp): A's differential contributions of the block
// grouped by target column.
void emit_bvt(const RowParts* rps, const RowMeta* meta, uint32_t nr, uint32_t B, uint64_t wlo, uint32_t W,
              std::vector<uint32_t>& so, std::vector<uint32_t>& far_cols, BvtStats& st) {
  constexpr uint32_t kUnit = kBvtUnitCodes, kMaxUnits = kBvtMaxUnits;
  // contributions grouped by target with flat arrays (counting sort for the
  // 2W window targets, a sort for the few far columns); codes k | minus << 15
  // stay in row order within a target
  const uint32_t W2 = 2 * W;
  thread_local std::vector<uint32_t> cnt;
  thread_local std::vector<uint16_t> flat;
  thread_local std::vector<std::pair<uint32_t, uint16_t>> far;
  cnt.assign(W2 + 1, 0);
  far.clear();
  auto near_t = [&](uint64_t col) { return (uint32_t)(col - wlo); };
  auto inwin = [&](uint64_t col) { return col >= wlo && col < wlo + W; };
  for (int pass = 0; pass < 2; ++pass) {
    auto put = [&](uint32_t t, uint32_t code) {
      if (pass == 0) ++cnt[t + 1];
      else flat[cnt[t]++] = (uint16_t)code;
    };
    for (uint32_t k = 0; k < nr; ++k) {
      const RowParts& rp = rps[k];
      for (uint32_t c : rp.minus) {
        if (inwin(c)) put(near_t(c), k | 0x8000u);
        else if (pass == 0) far.push_back({c, (uint16_t)(k | 0x8000u)});
      }
      for (uint32_t c : rp.res) {
        if (inwin(c)) put(near_t(c), k);
        else if (pass == 0) far.push_back({c, (uint16_t)k});
      }
      for (const auto& iv : rp.ints) {
        const uint64_t a0 = iv.first, e0 = (uint64_t)iv.first + iv.second;
        const uint64_t ia = std::max<uint64_t>(a0, wlo), ie = std::min<uint64_t>(e0, wlo + W);
        if (ia < ie) {  // in-window part: two difference entries
          put(W + near_t(ia), k);
          if (ie < wlo + W) put(W + near_t(ie), k | 0x8000u);
        }
        if (pass == 0)
          for (uint64_t c = a0; c < e0; ++c)  // out-of-window part: one far entry per column
            if (c < ia || c >= ie) far.push_back({(uint32_t)c, (uint16_t)k});
      }
    }
    if (pass == 0) {
      for (uint32_t t = 0; t < W2; ++t) cnt[t + 1] += cnt[t];
      flat.resize(cnt[W2] + far.size());
    } else {
      for (uint32_t t = W2; t > 0; --t) cnt[t] = cnt[t - 1];  // restore the starts
      cnt[0] = 0;
    }
  }
  std::sort(far.begin(), far.end());
  far_cols.clear();
  struct T {
    uint32_t target, start, count;
  };
  std::vector<T> targets;
  for (uint32_t t = 0; t < W2; ++t)
    if (cnt[t + 1] > cnt[t]) targets.push_back({t, cnt[t], cnt[t + 1] - cnt[t]});
  {
    uint32_t pos = cnt[W2];
    for (size_t q = 0; q < far.size();) {
      size_t e = q;
      const uint32_t start = pos;
      while (e < far.size() && far[e].first == far[q].first) flat[pos++] = far[e++].second;
      targets.push_back({W2 + (uint32_t)far_cols.size(), start, pos - start});
      far_cols.push_back(far[q].first);
      q = e;
    }
  }
  if (W2 + far_cols.size() > 0x3fffffffu) throw std::runtime_error("BV-T: too many targets in a block");
  // units: <= kUnit codes, balanced; 1 unit -> single slices, 2..32 -> multi, more -> heavy
  struct U {
    uint32_t target, start, count;
    bool primary;
  };
  std::vector<U> units;
  std::vector<uint32_t> singles;                       // unit index
  std::vector<std::pair<uint32_t, uint32_t>> multis;   // (first unit, #units)
  std::vector<const T*> heavy;
  for (const T& t : targets) {
    const uint32_t ne = t.count;
    st.entries += ne;
    const uint32_t nu = (ne + kUnit - 1) / kUnit;
    if (nu > kMaxUnits) {
      heavy.push_back(&t);
      continue;
    }
    const uint32_t first = (uint32_t)units.size();
    for (uint32_t j = 0; j < nu; ++j) {
      const uint32_t p0 = (uint32_t)((uint64_t)j * ne / nu), p1 = (uint32_t)((uint64_t)(j + 1) * ne / nu);
      units.push_back(U{t.target, t.start + p0, p1 - p0, j == 0});
    }
    if (nu == 1) singles.push_back(first);
    else multis.push_back({first, nu});
  }
  struct Slice {
    std::vector<const U*> lanes;
    bool multi;
    uint32_t maxnu = 1;  // most units of one target in the slice
  };
  std::vector<Slice> slices;
  auto load = [&](const std::pair<uint32_t, uint32_t>& r) {
    uint32_t m = 0;
    for (uint32_t q = 0; q < r.second; ++q) m = std::max(m, units[r.first + q].count);
    return m;
  };
  std::stable_sort(multis.begin(), multis.end(), [&](const auto& a, const auto& b) {
    if (load(a) != load(b)) return load(a) > load(b);
    return a.second > b.second;
  });
  for (const auto& r : multis) {
    size_t t = 0;
    while (t < slices.size() && slices[t].lanes.size() + r.second > 32) ++t;
    if (t == slices.size()) slices.push_back(Slice{{}, true});
    for (uint32_t q = 0; q < r.second; ++q) slices[t].lanes.push_back(&units[r.first + q]);
    slices[t].maxnu = std::max(slices[t].maxnu, r.second);
  }
  std::stable_sort(singles.begin(), singles.end(),
                   [&](uint32_t a, uint32_t b) { return units[a].count > units[b].count; });
  for (size_t a = 0; a < singles.size(); a += 32) {
    Slice sl{{}, false};
    for (size_t q = a; q < std::min(singles.size(), a + 32); ++q) sl.lanes.push_back(&units[singles[q]]);
    slices.push_back(std::move(sl));
  }
  const uint32_t nsl = (uint32_t)slices.size(), nh = (uint32_t)heavy.size();
  if (nsl > 0xffffu || nh > 0xffffu) throw std::runtime_error("BV-T: block too large");
  so.assign(kBvtHead + 2 * nsl, 0u);
  so[0] = nsl | (nh << 16);
  so[3] = (uint32_t)far_cols.size();
  // coefficient schedule: rows with children, deepest level first, each
  // entry k | children mask << 10 (bit r-1: row k + r references k)
  so[4] = (uint32_t)so.size();
  {
    std::vector<uint32_t> dep(nr), mask(nr, 0);
    uint32_t dmax = 0;
    for (uint32_t k = 0; k < nr; ++k) {
      const uint32_t r = meta[k].r;
      dep[k] = r ? dep[k - r] + 1 : 0;
      if (r) mask[k - r] |= 1u << (r - 1);
    }
    std::vector<std::vector<uint32_t>> lv;
    for (uint32_t k = 0; k < nr; ++k)
      if (mask[k]) {
        if (dep[k] >= lv.size()) lv.resize(dep[k] + 1);
        lv[dep[k]].push_back(k | (mask[k] << 10));
        dmax = std::max(dmax, dep[k] + 1);
      }
    so.push_back(dmax);
    uint32_t acc = 0;
    for (uint32_t d = dmax; d-- > 0;) {  // level starts, processing order
      so.push_back(acc);
      acc += (uint32_t)lv[d].size();
    }
    so.push_back(acc);
    for (uint32_t d = dmax; d-- > 0;) so.insert(so.end(), lv[d].begin(), lv[d].end());
  }
  so[5] = (uint32_t)so.size();
  so.insert(so.end(), far_cols.begin(), far_cols.end());
  const uint32_t zc = B;  // padding code: the zero coefficient
  for (uint32_t s = 0; s < nsl; ++s) {
    const Slice& sl = slices[s];
    so[kBvtHead + 2 * s] = (uint32_t)so.size();
    uint32_t mne = 0;
    for (const U* u : sl.lanes) {
      mne = std::max<uint32_t>(mne, u->count);
      st.lane_iters_used += u->count;
    }
    uint32_t rounds = 0;
    while ((1u << rounds) < sl.maxnu) ++rounds;
    so.push_back(make_tmeta(mne, sl.multi, rounds));
    so[kBvtHead + 2 * s + 1] = so.back();  // the table repeats the meta word
    for (size_t l = 0; l < 32; ++l) so.push_back(l < sl.lanes.size() ? make_th(sl.lanes[l]->primary, sl.lanes[l]->target) : 0u);
    const uint32_t mnw = (mne + 1) / 2;
    const size_t b0 = so.size();
    so.resize(b0 + (size_t)mnw * 32, 0u);
    for (size_t l = 0; l < 32; ++l) {
      const U* u = l < sl.lanes.size() ? sl.lanes[l] : nullptr;
      for (uint32_t q = 0; q < mnw; ++q) {
        const uint32_t c0 = u && 2 * q < u->count ? flat[u->start + 2 * q] : zc;
        const uint32_t c1 = u && 2 * q + 1 < u->count ? flat[u->start + 2 * q + 1] : zc;
        so[b0 + (size_t)q * 32 + l] = (c0 << 16) | c1;
      }
    }
    st.lane_iters += 32ull * mne;
  }
  so[1] = (uint32_t)so.size();
  std::vector<uint32_t> hc;
  for (const T* t : heavy) {
    so.push_back(t->target);
    so.push_back(t->count);
    so.push_back((uint32_t)hc.size());
    for (uint32_t q = 0; q < t->count; q += 2)
      hc.push_back(((uint32_t)flat[t->start + q] << 16) | (q + 1 < t->count ? flat[t->start + q + 1] : zc));
  }
  so[2] = (uint32_t)so.size();
  so.insert(so.end(), hc.begin(), hc.end());
  while (so.size() % 4) so.push_back(0u);
  st.slices += nsl;
  st.heavy_targets += nh;
  st.far_slots += far_cols.size();
}

std::atomic<long long> g_tim[4];

}  // namespace

BvdLayout build_bvd(const BvDecoded& dec, const BvParams& bp, const BvdOptions& opt) {
  const HostCsr& g = dec.csr;
  BvdLayout L;
  BvdDims& D = L.dims;
  const uint32_t B = opt.block_rows, W = opt.window;
  if (B == 0 || (B & (B - 1)) || B % bp.segment_rows || B > 1024)
    throw std::invalid_argument("block_rows must be a power of two <= 1024 and a multiple of the BV segment");
  if (W % 16 || W == 0 || W > 16384) throw std::invalid_argument("window must be a positive multiple of 16, at most 16384");
  if (bp.window > 7) throw std::invalid_argument("the device layout supports BV windows w <= 7");
  D.n = g.n;
  D.block_rows = B;
  D.window = W;
  D.min_interval = bp.min_interval;
  D.nblocks = (uint32_t)(((uint64_t)g.n + B - 1) / B);
  D.max_depth = 0;
  D.pad = 0;
  const uint32_t nb = D.nblocks;
  std::vector<BitWriter> bstream(nb);
  L.blocks.resize(nb);
  std::vector<uint64_t> bbits(nb, 0), badds(nb, 0), bcodes(nb, 0), bgath(nb, 0), bin(nb, 0);
  std::vector<uint32_t> bdepth(nb, 0);
  std::vector<std::vector<uint32_t>> sstream(nb);
  std::vector<BvsStats> bst(nb);
  std::vector<std::vector<uint32_t>> tstream(nb), tfar(nb), bfar(nb);
  std::vector<BvtStats> tst(nb);
  std::vector<std::vector<uint32_t>> fstream(nb);
  std::vector<BvfStats> fst(nb);
  L.fblocks.resize(nb);
  if (2 * W + kBvfSlots + 1 >= kBvfIdxMask) throw std::invalid_argument("window too large for the BV-F term index");
  parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
    std::vector<RowParts> rps(B);
    RowParts rp0;
    std::vector<uint32_t> plus, cols, depth(B), hdr(B), escs, eff_r(B);
    std::vector<RowMeta> meta(B);
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
      auto tA = std::chrono::steady_clock::now();
      // pass 1: split rows, collect gathered columns, choose the x-window
      for (uint32_t k = 0; k < nr; ++k) {
        const uint32_t i = r0 + k;
        uint32_t r = dec.ref_dist[i];
        if (r && k < r) throw std::runtime_error("BV-D: reference crosses a block");
        RowParts& rp = rps[k];
        split_row(g, i, r, bp.min_interval, rp, plus);
        if (r) {
          // the reference's keep rule (ref_matrix.hpp:63-65: a reference is
          // used only if it makes the row strictly shorter) applied to the
          // product's terms: BV picks references by bits, and a copy that
          // skips many entries can cost more adds than the plain row
          const uint64_t tref = rp.minus.size() + rp.res.size() + 2ull * rp.ints.size();
          RowParts& p0 = rp0;
          split_row(g, i, 0, bp.min_interval, p0, plus);
          if (p0.res.size() + 2ull * p0.ints.size() <= tref) {
            std::swap(rp, p0);
            r = 0;
          }
        }
        eff_r[k] = r;
        depth[k] = r ? depth[k - r] + 1 : 0;
        bdepth[b] = std::max(bdepth[b], depth[k]);
        for (auto& iv : rp.ints) {
          cols.push_back(iv.first);
          cols.push_back(iv.first + iv.second - 1);
        }
        for (uint32_t c : rp.minus) cols.push_back(c);
        for (uint32_t c : rp.res) cols.push_back(c);
      }
      radix_sort_u32(cols);
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
        const uint32_t r = eff_r[k];
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
        meta[k] = RowMeta{r, nm, ns, ni, wp, wl, far, body.nbits, 0};
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
        meta[k].nbits = body.nbits - meta[k].bit0;
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
      auto tB = std::chrono::steady_clock::now();
      if (opt.bvs) emit_bvs(rps.data(), meta.data(), body, nr, lo, W, bp.min_interval, sstream[b], bst[b]);
      if (opt.bvf) {
        // the shared host/device block builder (bvf_block.hpp)
        const BvfRowsView view{g.row_offsets.data(), g.cols.data(), dec.ref_dist.data(), g.n};
        uint64_t E = 0, Er = 0;
        for (uint32_t k = 0; k < nr; ++k) {
          const uint32_t i = r0 + k, r = dec.ref_dist[i];
          E += g.deg(i);
          if (r && k >= r) Er += g.deg(i - r);
        }
        thread_local std::vector<uint32_t> arena, obuf;
        arena.resize(bvf_block_scratch_words(E, Er, nr, bp.min_interval));
        obuf.assign(bvf_block_out_words(E, Er, nr, bp.min_interval), 0u);
        BvfArena ar{arena.data(), arena.size(), 0};
        const BvfBlockResult res = bvf_build_block(view, (uint32_t)b, B, W, bp.min_interval, ar, obuf.data(), obuf.size());
        if (res.err) throw std::runtime_error("BV-F block build failed (code " + std::to_string(res.err) + ")");
        fstream[b].assign(obuf.begin(), obuf.begin() + res.nwords);
        L.fblocks[b] = res.info;
        BvfStats& t = fst[b];
        t.terms = res.terms;
        t.pad_terms = res.pad_terms;
        t.slot_terms = res.slot_terms;
        t.esc_terms = res.esc_terms;
        t.esc_blocks = (res.info.flags & kBvfFlagEsc) ? 1 : 0;
        t.max_K = res.info.K;
        t.min_cbits = res.info.cbits;
        if (res.info.wlo != (uint32_t)lo || res.depth != bdepth[b] || res.adds != badds[b])
          throw std::runtime_error("BV-F block builder disagrees with the BV-D pass (window / depth / adds)");
      }
      auto tC = std::chrono::steady_clock::now();
      {  // columns this block reads outside its x-window (read set of a shard)
        std::vector<uint32_t>& fc = bfar[b];
        fc.clear();
        auto out = [&](uint64_t c) { return c < lo || c >= lo + W; };
        for (uint32_t k = 0; k < nr; ++k) {
          const RowParts& rp = rps[k];
          for (uint32_t c : rp.minus)
            if (out(c)) fc.push_back(c);
          for (uint32_t c : rp.res)
            if (out(c)) fc.push_back(c);
          for (const auto& iv : rp.ints)
            for (uint64_t c = iv.first; c < (uint64_t)iv.first + iv.second; ++c)
              if (out(c)) fc.push_back((uint32_t)c);
        }
        std::sort(fc.begin(), fc.end());
        fc.erase(std::unique(fc.begin(), fc.end()), fc.end());
      }
      auto tD = std::chrono::steady_clock::now();
      if (opt.bvt) emit_bvt(rps.data(), meta.data(), nr, B, lo, W, tstream[b], tfar[b], tst[b]);
      auto tE = std::chrono::steady_clock::now();
      g_tim[0] += std::chrono::duration_cast<std::chrono::microseconds>(tB - tA).count();
      g_tim[1] += std::chrono::duration_cast<std::chrono::microseconds>(tC - tB).count();
      g_tim[2] += std::chrono::duration_cast<std::chrono::microseconds>(tD - tC).count();
      g_tim[3] += std::chrono::duration_cast<std::chrono::microseconds>(tE - tD).count();
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
  // BV-S
  L.sblocks = L.blocks;
  uint64_t soff = 0;
  std::vector<uint32_t> ssz(nb);
  uint64_t hitems = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    L.sblocks[b].word_offset = soff;
    L.sblocks[b].nwords = (uint32_t)sstream[b].size();
    L.sblocks[b].nesc = 0;
    if (hitems > 0xffffffffull) throw std::runtime_error("BV-S: too many heavy-row work items");
    if (!sstream[b].empty()) sstream[b][3] = (uint32_t)hitems;  // the block's first heavy work item (global)
    hitems += bst[b].heavy_chunks;
    L.sstats.heavy_chunks += bst[b].heavy_chunks;
    soff += sstream[b].size();
    ssz[b] = (uint32_t)sstream[b].size();
    L.sstats.max_block_words = std::max(L.sstats.max_block_words, ssz[b]);
    L.sstats.slices += bst[b].slices;
    L.sstats.heavy_rows += bst[b].heavy_rows;
    L.sstats.lane_words += bst[b].lane_words;
    L.sstats.lane_words_used += bst[b].lane_words_used;
    L.sstats.lane_iters += bst[b].lane_iters;
    L.sstats.lane_iters_used += bst[b].lane_iters_used;
  }
  std::sort(ssz.begin(), ssz.end());
  L.sstats.p995_block_words = nb ? ssz[std::min<uint64_t>(nb - 1, (uint64_t)(nb * 0.995))] : 0;
  L.swords.assign(soff + 64, 0);  // guard words: lanes read one word past their slice
  parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
    for (uint64_t b = b0; b < b1; ++b)
      if (!sstream[b].empty())
        std::memcpy(L.swords.data() + L.sblocks[b].word_offset, sstream[b].data(), sstream[b].size() * 4);
  });
  L.sstats.stream_bytes = soff * 4;
  // BV-F
  {
    uint64_t foff = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      L.fblocks[b].word_offset = foff;
      foff += fstream[b].size();
      const BvfStats& t = fst[b];
      BvfStats& a = L.fstats;
      a.terms += t.terms;
      a.pad_terms += t.pad_terms;
      a.slot_terms += t.slot_terms;
      a.esc_terms += t.esc_terms;
      a.esc_blocks += t.esc_blocks;
      a.max_K = std::max(a.max_K, t.max_K);
      a.min_cbits = std::min(a.min_cbits, t.min_cbits);
    }
    L.fwords.assign(foff + 64, 0);  // guard words
    parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
      for (uint64_t b = b0; b < b1; ++b)
        if (!fstream[b].empty())
          std::memcpy(L.fwords.data() + L.fblocks[b].word_offset, fstream[b].data(), fstream[b].size() * 4);
    });
    L.fstats.stream_bytes = foff * 4;
  }
  // per-block out-of-window read columns
  L.rfar_ptr.assign(nb + 1, 0);
  for (uint32_t b = 0; b < nb; ++b) L.rfar_ptr[b + 1] = L.rfar_ptr[b] + bfar[b].size();
  L.rfar.resize(L.rfar_ptr[nb]);
  for (uint32_t b = 0; b < nb; ++b) std::copy(bfar[b].begin(), bfar[b].end(), L.rfar.begin() + L.rfar_ptr[b]);
  // BV-T + combine tables
  L.tblocks = L.blocks;
  uint64_t toff = 0, fslot = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    L.tblocks[b].word_offset = toff;
    L.tblocks[b].nwords = (uint32_t)tstream[b].size();
    L.tblocks[b].nesc = 0;
    L.tblocks[b].pad[0] = (uint32_t)fslot;
    toff += tstream[b].size();
    fslot += tfar[b].size();
    L.tstats.slices += tst[b].slices;
    L.tstats.heavy_targets += tst[b].heavy_targets;
    L.tstats.far_slots += tst[b].far_slots;
    L.tstats.entries += tst[b].entries;
    L.tstats.lane_iters += tst[b].lane_iters;
    L.tstats.lane_iters_used += tst[b].lane_iters_used;
  }
  if (fslot > 0xffffffffull) throw std::runtime_error("BV-T: too many far slots");
  L.twords.assign(toff + 64, 0);
  parallel_for(nb, [&](uint64_t b0, uint64_t b1) {
    for (uint64_t b = b0; b < b1; ++b)
      if (!tstream[b].empty())
        std::memcpy(L.twords.data() + L.tblocks[b].word_offset, tstream[b].data(), tstream[b].size() * 4);
  });
  L.tstats.stream_bytes = toff * 4;
  {
    const uint64_t ntiles = nb;  // column tiles of block_rows columns (the matrix is square)
    std::vector<std::vector<uint32_t>> tb(ntiles);
    for (uint32_t b = 0; b < nb; ++b) {
      const uint64_t w0 = L.blocks[b].wlo, w1 = std::min<uint64_t>(g.n, w0 + W);
      if (w1 <= w0) continue;
      for (uint64_t t = w0 / B; t <= (w1 - 1) / B && t < ntiles; ++t) tb[t].push_back(b);
    }
    L.tile_ptr.assign(ntiles + 1, 0);
    for (uint64_t t = 0; t < ntiles; ++t) L.tile_ptr[t + 1] = L.tile_ptr[t] + (uint32_t)tb[t].size();
    L.tile_blk.clear();
    for (auto& v : tb) L.tile_blk.insert(L.tile_blk.end(), v.begin(), v.end());
    std::vector<std::pair<uint32_t, uint32_t>> fp;
    fp.reserve(fslot);
    for (uint32_t b = 0; b < nb; ++b)
      for (size_t f = 0; f < tfar[b].size(); ++f) fp.push_back({tfar[b][f], L.tblocks[b].pad[0] + (uint32_t)f});
    std::sort(fp.begin(), fp.end());
    L.farp.resize(fp.size() * 2);
    L.farp_ptr.assign(ntiles + 1, 0);
    for (size_t q = 0; q < fp.size(); ++q) {
      L.farp[2 * q] = fp[q].first;
      L.farp[2 * q + 1] = fp[q].second;
      L.farp_ptr[fp[q].first / B + 1]++;
    }
    for (uint64_t t = 0; t < ntiles; ++t) L.farp_ptr[t + 1] += L.farp_ptr[t];
  }
  L.stats.block_table_bytes = (uint64_t)nb * sizeof(BvdBlockInfo);
  if (getenv("CMVG_BUILD_TIMING"))
    fprintf(stderr, "build_bvd thread-us: bvd %lld bvs %lld readset %lld bvt %lld\n", (long long)g_tim[0],
            (long long)g_tim[1], (long long)g_tim[2], (long long)g_tim[3]);
  return L;
}

}  // namespace cmvg
