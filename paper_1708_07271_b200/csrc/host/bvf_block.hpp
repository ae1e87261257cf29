// One BV-F block (layout.hpp) from the decoded rows of a BV stream: the same
// code runs on the host (the CPU layout builder, one block per task) and on
// the device (cmvg_create's device build, bvf_build.cu: one block per warp,
// lane 0), so the two layouts are identical by construction.
//
// Per row i of the block (reference include/cmv/ref_matrix.hpp:13-52: row i's
// A' row against its reference i - r): minus = the reference's entries the
// row lacks, plus = the row's entries the reference lacks, split into maximal
// runs >= Lmin (intervals) and residuals -- BV's own extra-list split; the
// reference is dropped when the plain row has no more terms (the keep rule,
// ref_matrix.hpp:63-65).  Then the block's x-window, far slots, the flat term
// list, the chunking, the bank schedule, escapes and the stream (layout.hpp).
//
// Working memory comes from a caller-provided arena (bump allocation, sized by
// bvf_block_scratch_words); no allocation, no standard library.
#pragma once
#include <cstdint>

#include "layout.hpp"

#ifdef __CUDACC__
#define CMVG_HD __host__ __device__
#else
#define CMVG_HD
#endif

namespace cmvg {

struct BvfRowsView {
  const uint64_t* ro;   // CSR row offsets (n + 1)
  const uint32_t* co;   // CSR columns (sorted, dedup'd per row)
  const uint8_t* ref;   // BV reference distance per row (0 = none)
  uint32_t n;
};

struct BvfBlockResult {
  BvfBlockInfo info;      // word_offset left 0
  uint32_t nwords;        // block stream words written
  uint32_t depth;         // longest reference chain in the block
  uint64_t adds;          // #refs + #minus + #residual + 2 #intervals (ref_matvec.hpp:11-18)
  uint64_t gathered;      // gathered columns (interval ends, minus, residuals)
  uint64_t in_window;     // ... of them inside the x-window
  uint32_t max_far;       // largest out-of-window column + 1 (0 = none)
  uint32_t max_deg;
  uint64_t terms, pad_terms, slot_terms, esc_terms;
  int err;                // 0 ok; 1 arena or output too small; 2 bad reference; 3 block too large
  uint64_t cyc[6];        // (device) clock cycles per phase: splits, window, far slots, terms, schedule, stream
};

CMVG_HD inline uint64_t bvfb_clock() {
#ifdef __CUDA_ARCH__
  return clock64();
#else
  return 0;
#endif
}

struct BvfArena {
  uint32_t* base;
  uint64_t cap, used;
  CMVG_HD uint32_t* take(uint64_t words) {
    words = (words + 3) & ~3ull;
    if (used + words > cap) return nullptr;
    uint32_t* p = base + used;
    used += words;
    return p;
  }
};

// arena words a block needs: E = the block's edges, Er = the edges of its
// rows' references (sum of deg(i - r_i) over rows with r_i != 0), nr rows.
// Bounds of every allocation bvf_build_block makes (4-word aligned): minus
// <= Er; a row's residual and interval entries <= its degree (<= E in all);
// intervals <= E / Lmin; terms <= minus + residuals + max(2, len) per
// interval + 2 pads per row <= Er + 2 E + 2 nr; far occurrences <= Er + E.
CMVG_HD inline uint64_t bvf_block_nmax(uint64_t E, uint64_t Er, uint32_t nr, uint32_t lmin) {
  (void)lmin;
  return Er + 2 * E + 2 * (uint64_t)nr + 16;
}
CMVG_HD inline uint64_t bvf_block_scratch_words(uint64_t E, uint64_t Er, uint32_t nr, uint32_t lmin) {
  const uint64_t ni = E / (lmin ? lmin : 1) + 1;
  const uint64_t ncols = 2 * ni + Er + E, nfar = Er + E;
  const uint64_t Nmax = bvf_block_nmax(E, Er, nr, lmin);
  const uint64_t Npad = Nmax + 16 * (Nmax / 4096 + 1);
  return 7 * ((uint64_t)nr + 1) + (Er + 1) + (E + 1) + 2 * (ni + 1) + 2 * (ncols + 1) + 260 + 2 * (nfar + 1) +
         (Npad / 2 + 2) + Npad + (Nmax + 1) + (Nmax / 2 + 2) + (Nmax + 1) + 4 * 32;
}
// output words a block needs (bound)
CMVG_HD inline uint64_t bvf_block_out_words(uint64_t E, uint64_t Er, uint32_t nr, uint32_t lmin) {
  const uint64_t Nmax = bvf_block_nmax(E, Er, nr, lmin);
  const uint64_t Npad = Nmax + 16 * (Nmax / 4096 + 1);
  return 132 + kBvfRnWords + 132 + (256 + 8) + Nmax + Npad / 2 + 64;
}

namespace bvfb {

template <typename T>
CMVG_HD inline T mn(T a, T b) { return a < b ? a : b; }
template <typename T>
CMVG_HD inline T mx(T a, T b) { return a > b ? a : b; }

// LSD radix sort of u32 keys (8-bit digits) with a temp buffer of n words
CMVG_HD inline void radix_u32(uint32_t* v, uint32_t* tmp, uint64_t n, uint32_t* cnt /* 257 */) {
  if (n < 2) return;
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 8 * pass;
    for (int d = 0; d < 257; ++d) cnt[d] = 0;
    for (uint64_t i = 0; i < n; ++i) ++cnt[((v[i] >> sh) & 255u) + 1];
    for (int d = 0; d < 256; ++d) cnt[d + 1] += cnt[d];
    for (uint64_t i = 0; i < n; ++i) tmp[cnt[(v[i] >> sh) & 255u]++] = v[i];
    for (uint64_t i = 0; i < n; ++i) v[i] = tmp[i];
  }
}

// split of row i against reference row i - r (r = 0: plain row) into
// minus / residual / interval lists; returns false on overflow of the caps
struct Split {
  uint32_t nm, ns, ni;
};
CMVG_HD inline Split split_row(const BvfRowsView& g, uint32_t i, uint32_t r, uint32_t lmin, uint32_t* minus,
                               uint32_t* res, uint32_t* ist, uint32_t* ilen, bool count_only) {
  Split sp{0, 0, 0};
  const uint32_t* L = g.co + g.ro[i];
  const uint32_t dl = (uint32_t)(g.ro[i + 1] - g.ro[i]);
  const uint32_t* R = r ? g.co + g.ro[i - r] : nullptr;
  const uint32_t dr = r ? (uint32_t)(g.ro[i - r + 1] - g.ro[i - r]) : 0u;
  uint32_t a = 0, b = 0;
  // the plus list is consumed on the fly: a pending run [rs, rs + rl)
  uint32_t rs = 0, rl = 0;
  auto flush = [&]() {
    if (!rl) return;
    if (rl >= lmin) {
      if (!count_only) {
        ist[sp.ni] = rs;
        ilen[sp.ni] = rl;
      }
      ++sp.ni;
    } else {
      if (!count_only)
        for (uint32_t t = 0; t < rl; ++t) res[sp.ns + t] = rs + t;
      sp.ns += rl;
    }
    rl = 0;
  };
  auto plus = [&](uint32_t c) {
    if (rl && c == rs + rl) {
      ++rl;
    } else {
      flush();
      rs = c;
      rl = 1;
    }
  };
  while (a < dl || b < dr) {
    if (b >= dr || (a < dl && L[a] < R[b])) {
      plus(L[a++]);
    } else if (a >= dl || R[b] < L[a]) {
      if (!count_only) minus[sp.nm] = R[b];
      ++sp.nm;
      ++b;
    } else {
      ++a;
      ++b;
    }
  }
  flush();
  return sp;
}

}  // namespace bvfb

// Builds block b into out[0, out_cap).  Returns the result (err != 0 on
// failure: the caller then treats the build as failed).
CMVG_HD inline BvfBlockResult bvf_build_block(const BvfRowsView& g, uint32_t b, uint32_t B, uint32_t W, uint32_t lmin,
                                              BvfArena& ar, uint32_t* out, uint64_t out_cap) {
  using namespace bvfb;
  BvfBlockResult R{};
  const uint32_t r0 = b * B, r1 = mn<uint32_t>(g.n, (uint32_t)((uint64_t)b * B + B));
  const uint32_t nr = r1 - r0;
  const uint32_t F0 = bvf_f0(W), ZERO = bvf_zero(W);
  auto fail = [&](int e) {
    R.err = e;
    return R;
  };
  uint64_t tc = bvfb_clock();
  auto tick = [&](int ph) {
    const uint64_t t = bvfb_clock();
    R.cyc[ph] += t - tc;
    tc = t;
  };
  // ---- per-row splits (capacities from the rows' degrees)
  uint64_t E = 0, Er = 0;
  uint32_t maxdeg = 0;
  for (uint32_t k = 0; k < nr; ++k) {
    const uint32_t i = r0 + k, r = g.ref[i];
    const uint32_t d = (uint32_t)(g.ro[i + 1] - g.ro[i]);
    E += d;
    maxdeg = mx(maxdeg, d);
    if (r) {
      if (k < r) return fail(2);  // a reference crosses the block
      Er += g.ro[i - r + 1] - g.ro[i - r];
    }
  }
  const uint64_t ni_cap = E / (lmin ? lmin : 1) + 1;
  uint32_t* eff = ar.take(nr);
  uint32_t* dep = ar.take(nr);
  uint32_t* mo = ar.take(nr + 1);
  uint32_t* so = ar.take(nr + 1);
  uint32_t* io = ar.take(nr + 1);
  uint32_t* mcol = ar.take(Er + 1);
  uint32_t* rcol = ar.take(E + 1);
  uint32_t* ist = ar.take(ni_cap + 1);
  uint32_t* ilen = ar.take(ni_cap + 1);
  if (!eff || !dep || !mo || !so || !io || !mcol || !rcol || !ist || !ilen) return fail(1);
  uint32_t nm = 0, ns = 0, nI = 0, depth = 0;
  uint64_t adds = 0;
  for (uint32_t k = 0; k < nr; ++k) {
    const uint32_t i = r0 + k;
    uint32_t r = g.ref[i];
    mo[k] = nm;
    so[k] = ns;
    io[k] = nI;
    Split sp = split_row(g, i, r, lmin, mcol + nm, rcol + ns, ist + nI, ilen + nI, false);
    if (r) {
      // the reference's keep rule applied to the product's terms
      const uint64_t tref = (uint64_t)sp.nm + sp.ns + 2ull * sp.ni;
      const Split p0 = split_row(g, i, 0, lmin, nullptr, nullptr, nullptr, nullptr, true);
      if ((uint64_t)p0.ns + 2ull * p0.ni <= tref) {
        sp = split_row(g, i, 0, lmin, mcol + nm, rcol + ns, ist + nI, ilen + nI, false);
        r = 0;
      }
    }
    eff[k] = r;
    dep[k] = r ? dep[k - r] + 1 : 0;
    depth = mx(depth, dep[k]);
    nm += sp.nm;
    ns += sp.ns;
    nI += sp.ni;
    adds += (r ? 1u : 0u) + sp.nm + sp.ns + 2ull * sp.ni;
  }
  mo[nr] = nm;
  so[nr] = ns;
  io[nr] = nI;
  R.depth = depth;
  R.adds = adds;
  R.max_deg = maxdeg;
  tick(0);
  // ---- the x-window: the W-column range holding most gathered columns
  const uint64_t ncols = 2ull * nI + nm + ns;
  uint32_t* cols = ar.take(ncols + 1);
  uint32_t* tmp = ar.take(ncols + 1);
  uint32_t* cnt = ar.take(260);
  if (!cols || !tmp || !cnt) return fail(1);
  {
    uint64_t q = 0;
    for (uint32_t t = 0; t < nI; ++t) {
      cols[q++] = ist[t];
      cols[q++] = ist[t] + ilen[t] - 1;
    }
    for (uint32_t t = 0; t < nm; ++t) cols[q++] = mcol[t];
    for (uint32_t t = 0; t < ns; ++t) cols[q++] = rcol[t];
  }
  radix_u32(cols, tmp, ncols, cnt);
  uint64_t best = 0, best_lo = r0;
  for (uint64_t a = 0, e = 0; a < ncols; ++a) {
    while (e < ncols && cols[e] < (uint64_t)cols[a] + W) ++e;
    if (e - a > best) {
      best = e - a;
      best_lo = cols[a];
    }
  }
  uint64_t lo = best_lo;
  if (ncols) {
    const uint64_t lim = mn<uint64_t>(best_lo + W, 0xffffffffull);
    uint64_t lb = 0, hb = ncols;  // lower_bound(cols, lim)
    while (lb < hb) {
      const uint64_t md = (lb + hb) / 2;
      if (cols[md] < lim) lb = md + 1;
      else hb = md;
    }
    const uint32_t hi = cols[lb - 1];
    const uint64_t slack = best_lo + W - 1 - hi;
    lo = best_lo >= slack / 2 ? best_lo - slack / 2 : 0;
  }
  lo &= ~15ull;
  const uint64_t wlo = lo;
  tick(1);
  auto inwin = [&](uint64_t c) { return c >= wlo && c < wlo + W; };
  auto int_inside = [&](uint32_t t) { return ist[t] >= wlo && (uint64_t)ist[t] + ilen[t] <= wlo + W; };
  {
    uint64_t in_cnt = 0;
    for (uint64_t q = 0; q < ncols; ++q) in_cnt += inwin(cols[q]) ? 1u : 0u;
    R.gathered = ncols;
    R.in_window = in_cnt;
  }
  // ---- far columns, the most used ones first into the slots
  uint64_t nfar = 0;
  for (uint32_t t = 0; t < nm; ++t) nfar += inwin(mcol[t]) ? 0u : 1u;
  for (uint32_t t = 0; t < ns; ++t) nfar += inwin(rcol[t]) ? 0u : 1u;
  for (uint32_t t = 0; t < nI; ++t)
    if (!int_inside(t))
      for (uint64_t c = ist[t]; c < (uint64_t)ist[t] + ilen[t]; ++c) nfar += inwin(c) ? 0u : 1u;
  uint32_t* farc = ar.take(nfar + 1);
  uint32_t* ftmp = ar.take(nfar + 1);
  if (!farc || !ftmp) return fail(1);
  {
    uint64_t q = 0;
    for (uint32_t t = 0; t < nm; ++t)
      if (!inwin(mcol[t])) farc[q++] = mcol[t];
    for (uint32_t t = 0; t < ns; ++t)
      if (!inwin(rcol[t])) farc[q++] = rcol[t];
    for (uint32_t t = 0; t < nI; ++t)
      if (!int_inside(t))
        for (uint64_t c = ist[t]; c < (uint64_t)ist[t] + ilen[t]; ++c)
          if (!inwin(c)) farc[q++] = (uint32_t)c;
  }
  radix_u32(farc, ftmp, nfar, cnt);
  R.max_far = nfar ? farc[nfar - 1] + 1u : 0u;
  // top kBvfSlots by (count desc, column asc): a sorted insertion list
  uint64_t topk[kBvfSlots];
  uint32_t ntop = 0;
  for (uint64_t a = 0; a < nfar;) {
    uint64_t e = a;
    while (e < nfar && farc[e] == farc[a]) ++e;
    const uint64_t key = ((uint64_t)(0xffffffffu - (uint32_t)(e - a)) << 32) | farc[a];
    if (ntop < kBvfSlots || key < topk[ntop - 1]) {
      uint32_t p = ntop < kBvfSlots ? ntop++ : ntop - 1;
      while (p > 0 && topk[p - 1] > key) {
        topk[p] = topk[p - 1];
        --p;
      }
      topk[p] = key;
    }
    a = e;
  }
  const uint32_t nslot = ntop;
  // slot lookup: (column, slot) sorted by column
  uint32_t scol[kBvfSlots], sidx[kBvfSlots];
  for (uint32_t s = 0; s < nslot; ++s) {
    const uint32_t c = (uint32_t)topk[s];
    uint32_t p = s;
    while (p > 0 && scol[p - 1] > c) {
      scol[p] = scol[p - 1];
      sidx[p] = sidx[p - 1];
      --p;
    }
    scol[p] = c;
    sidx[p] = s;
  }
  tick(2);
  // ---- terms in row order
  uint64_t Nmax = (uint64_t)nm + ns + 2ull * nr + 16;  // + max(2, len) per interval
  for (uint32_t t = 0; t < nI; ++t) Nmax += int_inside(t) ? 2u : ilen[t];
  const uint64_t Kmax = 16ull * mx<uint64_t>(1, (Nmax + 4095) / 4096);
  const uint64_t Npad = Nmax + Kmax;
  uint16_t* codes = reinterpret_cast<uint16_t*>(ar.take((Npad + 1) / 2 + 1));
  uint32_t* ecol = ar.take(Npad);
  uint32_t* rstart = ar.take(nr + 1);
  if (!codes || !ecol || !rstart) return fail(1);
  uint64_t N = 0, slot_terms = 0, esc_terms = 0, pad_terms = 0, terms = 0, umax = 0;
  auto xterm = [&](uint32_t c, bool minus) {
    uint32_t code;
    if (inwin(c)) {
      code = (uint32_t)(c - wlo);
    } else {
      uint32_t lb = 0, hb = nslot;
      while (lb < hb) {
        const uint32_t md = (lb + hb) / 2;
        if (scol[md] < c) lb = md + 1;
        else hb = md;
      }
      if (lb < nslot && scol[lb] == c) {
        code = W + sidx[lb];
        ++slot_terms;
      } else {
        code = kBvfEsc;
        ++esc_terms;
      }
    }
    codes[N] = (uint16_t)(code | (minus ? kBvfMinus : 0u));
    ecol[N] = c;
    ++N;
    ++terms;
  };
  for (uint32_t k = 0; k < nr; ++k) {
    rstart[k] = (uint32_t)N;
    uint64_t u = (uint64_t)(mo[k + 1] - mo[k]) + (so[k + 1] - so[k]);
    for (uint32_t t = mo[k]; t < mo[k + 1]; ++t) xterm(mcol[t], true);
    for (uint32_t t = so[k]; t < so[k + 1]; ++t) xterm(rcol[t], false);
    for (uint32_t t = io[k]; t < io[k + 1]; ++t) {
      u += ilen[t];
      if (int_inside(t)) {
        const uint32_t a = (uint32_t)(ist[t] - wlo);
        codes[N] = (uint16_t)(F0 + a + ilen[t]);
        ecol[N++] = 0;
        codes[N] = (uint16_t)((F0 + a) | kBvfMinus);
        ecol[N++] = 0;
        terms += 2;
      } else {
        for (uint64_t c = ist[t]; c < (uint64_t)ist[t] + ilen[t]; ++c) xterm((uint32_t)c, false);
      }
    }
    // every row gets an even number (>= 2) of terms: rows end only on a
    // code word's high term
    while (N == rstart[k] || ((N - rstart[k]) & 1u)) {
      codes[N] = (uint16_t)ZERO;
      ecol[N++] = 0;
      ++pad_terms;
    }
    codes[N - 1] |= (uint16_t)kBvfEnd;
    umax = mx(umax, u);
  }
  rstart[nr] = (uint32_t)N;
  const uint32_t K = 16u * (uint32_t)mx<uint64_t>(1, (N + 4095) / 4096);
  if (K > 0xffffu || K > kBvfIdxMask) return fail(3);
  const uint32_t nact = (uint32_t)((N + K - 1) / K);
  pad_terms += (uint64_t)nact * K - N;
  for (uint64_t q = N; q < (uint64_t)nact * K; ++q) {
    codes[q] = (uint16_t)ZERO;
    ecol[q] = 0;
  }
  tick(3);
  // ---- bank schedule (layout.hpp; host/bvd_layout.cpp, bvf_schedule_terms):
  // in term step j the 32 chunks of a warp load table entries at once, in two
  // half-warp phases of 16 lanes; a row's terms may be summed in any order, so
  // each row's terms are re-dealt to the row's positions, most constrained
  // lane first, each taking the term whose bank pair (index mod 16) is least
  // loaded in its phase (an entry already loaded is free); F terms also count
  // their F lo load.  Ties go to the term whose 16-byte bank group (index mod
  // 8) is least loaded in the lane's quarter warp: the phase of the
  // multi-vector kernel's 16-byte table loads (cuda/bvf_matmat.cuh).
  {
    uint32_t* rowof = ar.take(N + 1);
    uint16_t* pc = reinterpret_cast<uint16_t*>(ar.take((N + 1) / 2 + 1));
    uint32_t* pe = ar.take(N + 1);
    uint32_t* pend = ar.take(nr + 1);
    if (!rowof || !pc || !pe || !pend) return fail(1);
    for (uint32_t k = 0; k < nr; ++k)
      for (uint32_t p = rstart[k]; p < rstart[k + 1]; ++p) rowof[p] = k;
    for (uint64_t q = 0; q < N; ++q) {
      pc[q] = (uint16_t)(codes[q] & ~kBvfEnd);
      pe[q] = ecol[q];
    }
    for (uint32_t k = 0; k < nr; ++k) pend[k] = rstart[k + 1];
    uint32_t lanes[16];
    uint16_t seen[16][8], fseen[16][8];
    uint8_t nseen[16], nfseen[16], qseen[16];  // qseen: per quarter warp, per 16-byte bank group
    for (uint32_t j = 0; j < K; ++j) {
      for (uint32_t h0 = 0; h0 < nact; h0 += 16) {
        uint32_t nl = 0;
        uint32_t lrow[16], lkey[16];
        for (uint32_t t = h0; t < mn(nact, h0 + 16); ++t)
          if ((uint64_t)t * K + j < N) {
            const uint32_t k = rowof[(uint64_t)t * K + j];
            lanes[nl] = t;
            lrow[nl] = k;
            lkey[nl++] = pend[k] - rstart[k];
          }
        // most constrained (fewest remaining terms) first; stable
        for (uint32_t a = 1; a < nl; ++a) {
          const uint32_t v = lanes[a], rv = lrow[a], kv = lkey[a];
          uint32_t p = a;
          while (p > 0 && kv < lkey[p - 1]) {
            lanes[p] = lanes[p - 1];
            lrow[p] = lrow[p - 1];
            lkey[p] = lkey[p - 1];
            --p;
          }
          lanes[p] = v;
          lrow[p] = rv;
          lkey[p] = kv;
        }
        for (int q = 0; q < 16; ++q) nseen[q] = nfseen[q] = qseen[q] = 0;
        uint32_t nf = 0;
        for (uint32_t q = 0; q < nl; ++q) {
          const uint64_t pos = (uint64_t)lanes[q] * K + j;
          const uint32_t k = lrow[q];
          uint8_t* qs = qseen + (((lanes[q] - h0) >> 3) << 3);
          uint32_t best_i = rstart[k], bcost = 0xffffffffu;
          bool bdup = false;
          for (uint32_t i = rstart[k]; i < pend[k]; ++i) {
            const uint32_t c = pc[i];
            uint32_t cost = 0;
            bool dup = true;
            if (!(c & kBvfEsc)) {
              const uint32_t idx = c & kBvfIdxMask, bk = idx & 15u;
              cost = nseen[bk];
              dup = false;
              for (uint32_t s = 0; s < mn<uint32_t>(nseen[bk], 8); ++s)
                if (seen[bk][s] == idx) {
                  cost = 0;
                  dup = true;
                }
              if (idx >= F0) {
                uint32_t fc = nfseen[bk];
                for (uint32_t s = 0; s < mn<uint32_t>(nfseen[bk], 8); ++s)
                  if (fseen[bk][s] == idx) fc = 0;
                cost += fc + (nf == 0 ? 1u : 0u);
              }
              cost = cost * 64u + (dup ? 0u : qs[idx & 7u]);
            }
            if (cost < bcost) {
              bcost = cost;
              best_i = i;
              bdup = dup;
              if (!cost) break;
            }
          }
          const uint16_t c = pc[best_i];
          const uint32_t e = pe[best_i];
          --pend[k];
          pc[best_i] = pc[pend[k]];
          pe[best_i] = pe[pend[k]];
          codes[pos] = c;
          ecol[pos] = e;
          if (!bdup && !(c & kBvfEsc)) ++qs[c & 7u];
          if (!bdup) {
            const uint32_t bk = (c & kBvfIdxMask) & 15u;
            if (nseen[bk] < 8) seen[bk][nseen[bk]] = (uint16_t)(c & kBvfIdxMask);
            ++nseen[bk];
          }
          if (!(c & kBvfEsc) && (c & kBvfIdxMask) >= F0) {
            const uint32_t idx = c & kBvfIdxMask, bk = idx & 15u;
            bool have = false;
            for (uint32_t s = 0; s < mn<uint32_t>(nfseen[bk], 8); ++s) have = have || fseen[bk][s] == idx;
            if (!have) {
              if (nfseen[bk] < 8) fseen[bk][nfseen[bk]] = (uint16_t)idx;
              ++nfseen[bk];
            }
            ++nf;
          }
        }
      }
    }
    for (uint32_t k = 0; k < nr; ++k) codes[rstart[k + 1] - 1] |= (uint16_t)kBvfEnd;  // a row's last position ends it
  }
  tick(4);
  // ---- escape terms: counted here, ordered and indexed with the stream below
  uint32_t nesc = 0;
  for (uint64_t i = 0; i < (uint64_t)nact * K; ++i) nesc += (codes[i] & kBvfEsc) ? 1u : 0u;
  // split grid: 2^cbits units per |x| <= 2^E, sums exact while < 2^53
  const uint64_t bound = 2ull * W + umax + 2ull * maxdeg + 2;
  uint32_t lg = 0;
  while ((1ull << lg) < bound) ++lg;
  const uint32_t cbits = (uint32_t)mx(8, mn(40, 51 - (int)lg));
  // ---- stream
  uint64_t o = 0;
  auto put = [&](uint32_t v) {
    if (o < out_cap) out[o] = v;
    ++o;
  };
  auto align4 = [&]() {
    while (o & 3u) put(0u);
  };
  // u16 first row of each chunk
  for (uint32_t t = 0; t < bvf_rn_off(nact); ++t) put(0u);
  for (uint32_t t = 0; t < nact; ++t) {
    const uint64_t i = (uint64_t)t * K;
    uint32_t lb = 0, hb = nr + 1;  // upper_bound(rstart[0, nr], i) - 1
    while (lb < hb) {
      const uint32_t md = (lb + hb) / 2;
      if (rstart[md] <= i) lb = md + 1;
      else hb = md;
    }
    const uint32_t row = mn(lb - 1, nr - 1);
    if (o <= out_cap) {
      const uint64_t w = t / 2;
      if (w < out_cap) out[w] |= (row & 0xffffu) << (16 * (t & 1));
    }
  }
  for (uint32_t t = 0; t < kBvfRnWords; ++t) put(0u);
  for (uint32_t k = 0; k < nr; ++k) {
    const uint64_t w = bvf_rn_off(nact) + (k >> 3);
    if (w < out_cap) out[w] |= (eff[k] & 15u) << (4 * (k & 7));
  }
  for (uint32_t s = 0; s < nslot; ++s) put((uint32_t)topk[s]);
  align4();
  const uint32_t esc_off = (uint32_t)o;
  if (nesc) {
    // The x values of a block's escapes are gathered ahead into one list; a
    // term holds its value's index relative to its chunk's start.  The 32
    // chunks of a warp are interleaved: their escapes are ordered by term
    // position, then lane, so the lanes of a warp (in lockstep over the term
    // positions) load adjacent values -- whole sectors instead of one value
    // per sector.  A chunk's start is the place of its first escape; a group
    // whose list would outgrow the 13-bit index keeps chunk-major order.
    for (uint32_t t = 0; t <= nact; ++t) put(0u);
    align4();
    const uint64_t col0 = o;
    uint32_t p = 0;
    for (uint32_t t0 = 0; t0 < nact; t0 += 32) {
      const uint32_t t1 = mn<uint32_t>(t0 + 32, nact);
      uint32_t gt = 0;
      for (uint64_t i = (uint64_t)t0 * K; i < (uint64_t)t1 * K; ++i) gt += (codes[i] & kBvfEsc) ? 1u : 0u;
      if (!gt) continue;
      uint32_t gstart[32];
      if (gt <= kBvfIdxMask + 1u) {
        uint32_t seen = 0;
        for (uint32_t i = 0; i < K; ++i)
          for (uint32_t t = t0; t < t1; ++t) {
            const uint64_t ci = (uint64_t)t * K + i;
            if (!(codes[ci] & kBvfEsc)) continue;
            if (!((seen >> (t - t0)) & 1u)) {
              seen |= 1u << (t - t0);
              gstart[t - t0] = p;
              if (esc_off + t < out_cap) out[esc_off + t] = p;
            }
            codes[ci] = (uint16_t)((codes[ci] & ~kBvfIdxMask) | (p - gstart[t - t0]));
            if (col0 + p < out_cap) out[col0 + p] = ecol[ci];
            ++p;
          }
      } else {
        for (uint32_t t = t0; t < t1; ++t) {
          if (esc_off + t < out_cap) out[esc_off + t] = p;
          uint32_t loc = 0;
          for (uint64_t ci = (uint64_t)t * K; ci < (uint64_t)(t + 1) * K; ++ci)
            if (codes[ci] & kBvfEsc) {
              codes[ci] = (uint16_t)((codes[ci] & ~kBvfIdxMask) | loc++);
              if (col0 + p < out_cap) out[col0 + p] = ecol[ci];
              ++p;
            }
        }
      }
    }
    if (esc_off + nact < out_cap) out[esc_off + nact] = p;  // the total
    o = col0 + p;
    align4();
  }
  const uint32_t codes_off = (uint32_t)o;
  for (uint32_t q = 0; q < K / 2; ++q)
    for (uint32_t t = 0; t < nact; ++t)
      put((uint32_t)codes[(uint64_t)t * K + 2 * q] | ((uint32_t)codes[(uint64_t)t * K + 2 * q + 1] << 16));
  align4();
  if (o > out_cap) return fail(1);
  R.nwords = (uint32_t)o;
  BvfBlockInfo& info = R.info;
  info.word_offset = 0;
  info.wlo = (uint32_t)wlo;
  info.K = (uint16_t)K;
  info.nact = (uint16_t)nact;
  info.nslot = (uint16_t)nslot;
  info.cbits = (uint8_t)cbits;
  info.flags = nesc ? kBvfFlagEsc : 0u;
  info.codes_off = codes_off;
  info.esc_off = esc_off;
  info.nwords = (uint32_t)o;
  tick(5);
  R.terms = terms;
  R.pad_terms = pad_terms;
  R.slot_terms = slot_terms;
  R.esc_terms = esc_terms;
  return R;
}

}  // namespace cmvg
