// Seeded synthetic graph generators for BASELINE.json configs 1-5
// (resolution of the spec gaps: SURVEY.md Appendix A).
//
// Determinism: every random draw comes from a counter-based stream keyed by
// (seed, row), so output is independent of the thread count.  Copy sources
// are restricted to the row's generator segment, so segments generate in
// parallel.
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "host.hpp"

namespace cmvg {
namespace {

inline uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct RowRng {
  uint64_t s;
  RowRng(uint64_t seed, uint64_t row) {
    s = seed * 0xD1B54A32D192ED03ull + row * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    splitmix(s);
  }
  uint64_t next() { return splitmix(s); }
  double uni() { return (next() >> 11) * (1.0 / 9007199254740992.0); }  // [0,1)
  uint64_t below(uint64_t k) { return (uint64_t)(uni() * (double)k); }
  uint32_t poisson(double lam) {
    double L = std::exp(-lam), p = 1.0;
    uint32_t k = 0;
    do { ++k; p *= uni(); } while (p > L && k < 1000);
    return k - 1;
  }
  uint64_t geometric(double mean) {  // support {1,2,...}, mean `mean`
    double q = 1.0 - 1.0 / mean;
    double u = uni();
    if (u <= 0) u = 1e-300;
    return 1 + (uint64_t)std::floor(std::log(u) / std::log(q));
  }
};

void sort_unique(std::vector<uint32_t>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

// Generates rows [r0, r1) of the copy model, where r0 is a segment start.
void copy_model_rows(const CopyModelParams& p, double lambda, uint32_t r0, uint32_t r1,
                     std::vector<std::vector<uint32_t>>& rows) {
  std::vector<uint32_t> tmp;
  for (uint32_t i = r0; i < r1; ++i) {
    RowRng rng(p.seed, i);
    tmp.clear();
    if (rng.uni() < p.p_ref) {
      uint32_t r = 1 + (uint32_t)rng.below(p.ref_window);
      if (i >= r0 + r) {
        for (uint32_t s : rows[i - r - r0])
          if (rng.uni() < p.p_copy) tmp.push_back(s);
      }
    }
    uint32_t K = rng.poisson(lambda);
    for (uint32_t k = 0; k < K; ++k) {
      int64_t g = (int64_t)rng.geometric(p.gap_mean);
      int64_t c = (rng.next() & 1) ? (int64_t)i + g : (int64_t)i - g;
      if (c < 0) c = -c;
      if (c >= (int64_t)p.n) c = 2 * ((int64_t)p.n - 1) - c;
      if (c < 0) c = 0;
      if (c >= (int64_t)p.n) c = p.n - 1;
      if (rng.uni() < p.p_run) {
        uint32_t len = p.run_min + (uint32_t)rng.below(p.run_max - p.run_min + 1);
        for (uint32_t t = 0; t < len && c + t < p.n; ++t) tmp.push_back((uint32_t)(c + t));
      } else {
        tmp.push_back((uint32_t)c);
      }
    }
    sort_unique(tmp);
    rows[i - r0] = tmp;
  }
}

HostCsr assemble(uint32_t n, uint32_t seg, const std::function<void(uint32_t, uint32_t, std::vector<std::vector<uint32_t>>&)>& gen) {
  uint32_t nseg = (n + seg - 1) / seg;
  std::vector<std::vector<uint32_t>> degs(nseg);
  std::vector<std::vector<uint32_t>> cols(nseg);
  parallel_for(nseg, [&](uint64_t b, uint64_t e) {
    std::vector<std::vector<uint32_t>> rows;
    for (uint64_t s = b; s < e; ++s) {
      uint32_t r0 = (uint32_t)(s * seg), r1 = (uint32_t)std::min<uint64_t>(n, (s + 1) * seg);
      rows.assign(r1 - r0, {});
      gen(r0, r1, rows);
      size_t tot = 0;
      for (auto& r : rows) tot += r.size();
      degs[s].resize(r1 - r0);
      cols[s].reserve(tot);
      for (uint32_t k = 0; k < r1 - r0; ++k) {
        degs[s][k] = (uint32_t)rows[k].size();
        cols[s].insert(cols[s].end(), rows[k].begin(), rows[k].end());
      }
    }
  });
  HostCsr g;
  g.n = n;
  g.row_offsets.resize((size_t)n + 1);
  std::vector<uint64_t> seg_base(nseg + 1, 0);
  for (uint32_t s = 0; s < nseg; ++s) seg_base[s + 1] = seg_base[s] + cols[s].size();
  g.cols.resize(seg_base[nseg]);
  g.row_offsets[0] = 0;
  parallel_for(nseg, [&](uint64_t b, uint64_t e) {
    for (uint64_t s = b; s < e; ++s) {
      uint64_t off = seg_base[s];
      uint32_t r0 = (uint32_t)(s * seg);
      for (size_t k = 0; k < degs[s].size(); ++k) {
        off += degs[s][k];
        g.row_offsets[r0 + k + 1] = off;
      }
      std::memcpy(g.cols.data() + seg_base[s], cols[s].data(), cols[s].size() * sizeof(uint32_t));
      std::vector<uint32_t>().swap(cols[s]);
    }
  });
  return g;
}

}  // namespace

double calibrate_copy_model_lambda(const CopyModelParams& p) {
  // Stationary estimate: d = p_ref*p_copy*d + lam*(1-p_run + p_run*E[len]).
  double elen = 0.5 * (p.run_min + p.run_max);
  double lam = p.mean_degree * (1.0 - p.p_ref * p.p_copy) / ((1 - p.p_run) + p.p_run * elen);
  uint32_t pilot = std::min<uint32_t>(p.n, 1u << 17);
  uint32_t seg = std::min(p.gen_segment, pilot);
  for (int it = 0; it < 6; ++it) {
    uint64_t edges = 0;
    // pilot over the first `pilot` rows, in segments like the real run
    for (uint32_t r0 = 0; r0 < pilot; r0 += seg) {
      uint32_t r1 = std::min(pilot, r0 + seg);
      std::vector<std::vector<uint32_t>> rows(r1 - r0);
      copy_model_rows(p, lam, r0, r1, rows);
      for (auto& r : rows) edges += r.size();
    }
    double mean = (double)edges / pilot;
    if (mean <= 0) break;
    double ratio = p.mean_degree / mean;
    lam *= ratio;
    if (std::fabs(ratio - 1) < 0.002) break;
  }
  return lam;
}

HostCsr generate_copy_model(const CopyModelParams& p) {
  if (p.n == 0) return HostCsr{0, {0}, {}};
  double lam = p.lambda > 0 ? p.lambda : calibrate_copy_model_lambda(p);
  return assemble(p.n, p.gen_segment, [&](uint32_t r0, uint32_t r1, std::vector<std::vector<uint32_t>>& rows) {
    copy_model_rows(p, lam, r0, r1, rows);
  });
}

HostCsr generate_social(const SocialParams& p) {
  // shifted Zipf P(d) ~ (d + shift)^-exponent on [deg_min, deg_max]
  std::vector<double> cdf(p.deg_max - p.deg_min + 1);
  double acc = 0;
  for (uint32_t d = p.deg_min; d <= p.deg_max; ++d) {
    acc += std::pow((double)d + p.zipf_shift, -p.zipf_exponent);
    cdf[d - p.deg_min] = acc;
  }
  for (auto& c : cdf) c /= acc;
  return assemble(p.n, p.gen_segment, [&](uint32_t r0, uint32_t r1, std::vector<std::vector<uint32_t>>& rows) {
    std::vector<uint32_t> tmp;
    for (uint32_t i = r0; i < r1; ++i) {
      RowRng rng(p.seed, i);
      double u = rng.uni();
      uint32_t d = p.deg_min + (uint32_t)(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      if (d > p.n) d = p.n;
      tmp.clear();
      if (rng.uni() < p.p_ref) {
        uint32_t r = 1 + (uint32_t)rng.below(p.ref_window);
        if (i >= r0 + r)
          for (uint32_t s : rows[i - r - r0])
            if (rng.uni() < p.p_copy) tmp.push_back(s);
      }
      if (tmp.size() > d) {  // keep a random d-subset of the copied successors
        for (uint32_t k = 0; k < d; ++k) std::swap(tmp[k], tmp[k + rng.below(tmp.size() - k)]);
        tmp.resize(d);
      }
      uint32_t cbase = i - i % p.community;
      uint32_t csize = std::min<uint32_t>(p.community, p.n - cbase);
      for (int round = 0; round < 6 && tmp.size() < d; ++round) {
        size_t need = d - tmp.size();
        for (size_t k = 0; k < need + need / 8 + 1; ++k) {
          if (rng.uni() < p.p_community) tmp.push_back(cbase + (uint32_t)rng.below(csize));
          else tmp.push_back((uint32_t)rng.below(p.n));
        }
        sort_unique(tmp);
        if (tmp.size() > d) {
          // drop a random surplus so the row has exactly d successors
          for (size_t k = 0; k < d; ++k) std::swap(tmp[k], tmp[k + rng.below(tmp.size() - k)]);
          tmp.resize(d);
        }
      }
      sort_unique(tmp);
      rows[i - r0] = tmp;
    }
  });
}

}  // namespace cmvg
