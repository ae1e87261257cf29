// Biclique covers: the paper's second
// computation-friendly format ("decompose the edges of G
// into a number of bicliques"), behind the reference's interface
// (include/cmv/biclique.hpp):
//   * extract_greedy  (biclique.hpp:48-61): deterministic greedy extraction;
//   * verify_cover    (biclique.hpp:63-64): exact, edge-disjoint coverage;
//   * compressed_size (biclique.hpp:33-34): sum |S_r| + |C_r| + |residual|;
//   * the BCV1 text container (biclique.hpp:66-73);
//   * the device layout of the product (csrc/bicover.cu): two CSR operands,
//     T (bicliques x targets) and M (rows x [residual columns | n + r for
//     every biclique r the row is a source of]), so y = M [x ; T x].
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <sstream>

#include "host.hpp"

namespace cmvg {

uint64_t BicliqueCover::compressed_size() const {
  uint64_t s = residual.size();
  for (const Biclique& b : bicliques) s += b.sources.size() + b.targets.size();
  return s;
}

namespace {

inline uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Candidate {
  uint64_t gain;
  std::vector<uint32_t> S, C;
};

bool contains_all(const std::vector<uint32_t>& row, const std::vector<uint32_t>& C) {
  return std::includes(row.begin(), row.end(), C.begin(), C.end());
}

void erase_sorted(std::vector<uint32_t>& v, uint32_t x) {
  auto it = std::lower_bound(v.begin(), v.end(), x);
  if (it != v.end() && *it == x) v.erase(it);
}

}  // namespace

// Greedy extraction (biclique.hpp:48-61).  A round hashes
// every row's remaining adjacency set with three min-hash seeds, buckets rows
// by signature, intersects each pair of bucket neighbours (in row order) to
// propose a target set C (|C| >= 2), expands the sources to every row whose
// remaining adjacency still contains C (via the in-list of C's rarest
// target), and scores gain = |S||C| - |S| - |C|.  The round emits the best
// candidate (ties: smaller S, then C, lexicographically) -- or, with
// per_round = 0, every candidate in that order that is still valid against
// the edges removed so far this round (a tractable mode for large graphs) --
// and removes its edges.  Stops when no candidate gains >= min_gain or after
// max_rounds rounds; the remaining edges become the residual.  Deterministic.
BicliqueCover extract_greedy(const HostCsr& g, uint64_t min_gain, uint64_t max_rounds, uint32_t per_round) {
  if (min_gain < 1) throw std::invalid_argument("extract_greedy: min_gain must be >= 1");
  const uint32_t n = g.n;
  std::vector<std::vector<uint32_t>> adj(n), inadj(n);
  for (uint32_t u = 0; u < n; ++u) {
    adj[u].assign(g.row(u), g.row(u) + g.deg(u));
    for (uint32_t j : adj[u]) inadj[j].push_back(u);  // ascending u: in-lists sorted
  }
  BicliqueCover cover;
  cover.n = n;
  std::vector<std::pair<uint64_t, uint32_t>> sig;
  for (uint64_t round = 0; round < max_rounds; ++round) {
    std::vector<Candidate> cands;
    for (uint64_t seed = 1; seed <= 3; ++seed) {
      sig.clear();
      for (uint32_t u = 0; u < n; ++u) {
        if (adj[u].size() < 2) continue;
        uint64_t h = ~0ull;
        for (uint32_t j : adj[u]) h = std::min(h, mix64(((uint64_t)j << 8) ^ seed));
        sig.emplace_back(h, u);
      }
      std::sort(sig.begin(), sig.end());
      for (size_t a = 0; a + 1 < sig.size(); ++a) {
        if (sig[a].first != sig[a + 1].first) continue;
        const uint32_t u = sig[a].second, v = sig[a + 1].second;
        Candidate c;
        std::set_intersection(adj[u].begin(), adj[u].end(), adj[v].begin(), adj[v].end(), std::back_inserter(c.C));
        if (c.C.size() < 2) continue;
        uint32_t rare = c.C[0];
        for (uint32_t j : c.C)
          if (inadj[j].size() < inadj[rare].size()) rare = j;
        for (uint32_t w : inadj[rare])
          if (contains_all(adj[w], c.C)) c.S.push_back(w);
        const uint64_t s = c.S.size(), t = c.C.size();
        if (s * t <= s + t || s * t - s - t < min_gain) continue;
        c.gain = s * t - s - t;
        cands.push_back(std::move(c));
      }
    }
    if (cands.empty()) break;
    std::sort(cands.begin(), cands.end(), [](const Candidate& a, const Candidate& b) {
      if (a.gain != b.gain) return a.gain > b.gain;
      if (a.S != b.S) return a.S < b.S;
      return a.C < b.C;
    });
    uint32_t emitted = 0;
    for (size_t q = 0; q < cands.size(); ++q) {
      if (q > 0 && cands[q].S == cands[q - 1].S && cands[q].C == cands[q - 1].C) continue;  // duplicate proposal
      Candidate& c = cands[q];
      if (emitted) {  // re-validate against this round's removals
        std::vector<uint32_t> S2;
        for (uint32_t w : c.S)
          if (contains_all(adj[w], c.C)) S2.push_back(w);
        const uint64_t s = S2.size(), t = c.C.size();
        if (s * t <= s + t || s * t - s - t < min_gain) continue;
        c.S.swap(S2);
      }
      for (uint32_t w : c.S)
        for (uint32_t j : c.C) {
          erase_sorted(adj[w], j);
          erase_sorted(inadj[j], w);
        }
      cover.bicliques.push_back(Biclique{c.S, c.C});
      ++emitted;
      if (per_round && emitted >= per_round) break;
    }
    if (!emitted) break;
  }
  for (uint32_t u = 0; u < n; ++u)
    for (uint32_t j : adj[u]) cover.residual.emplace_back(u, j);
  return cover;
}

// Structural invariants of a cover on its own (ids in range, sides sorted,
// strictly increasing and non-empty, residual sorted without duplicates).
void validate_cover_structure(const BicliqueCover& c) {
  for (size_t r = 0; r < c.bicliques.size(); ++r) {
    const Biclique& b = c.bicliques[r];
    if (b.sources.empty() || b.targets.empty()) throw std::invalid_argument("biclique cover: empty side");
    for (const auto* side : {&b.sources, &b.targets}) {
      for (size_t i = 0; i < side->size(); ++i) {
        if ((*side)[i] >= c.n) throw std::out_of_range("biclique cover: vertex id out of range");
        if (i && (*side)[i] <= (*side)[i - 1]) throw std::invalid_argument("biclique cover: ids not strictly ascending");
      }
    }
  }
  for (size_t i = 0; i < c.residual.size(); ++i) {
    if (c.residual[i].first >= c.n || c.residual[i].second >= c.n)
      throw std::out_of_range("biclique cover: residual edge out of range");
    if (i && c.residual[i] <= c.residual[i - 1])
      throw std::invalid_argument("biclique cover: residual not sorted / duplicate edge");
  }
}

// verify_cover (biclique.hpp:63-64): the biclique edge sets and the residual
// are pairwise disjoint and their union is exactly g's edge set.
bool verify_cover(const BicliqueCover& c, const HostCsr& g) {
  if (c.n != g.n) return false;
  try {
    validate_cover_structure(c);
  } catch (const std::exception&) {
    return false;
  }
  uint64_t covered = c.residual.size();
  for (const Biclique& b : c.bicliques) covered += (uint64_t)b.sources.size() * b.targets.size();
  if (covered != g.m()) return false;  // with the per-edge checks below: disjoint and exact
  std::vector<std::vector<uint32_t>> seen(g.n);
  for (const Biclique& b : c.bicliques)
    for (uint32_t u : b.sources) seen[u].insert(seen[u].end(), b.targets.begin(), b.targets.end());
  for (const auto& e : c.residual) seen[e.first].push_back(e.second);
  for (uint32_t u = 0; u < g.n; ++u) {
    std::vector<uint32_t>& s = seen[u];
    if (s.size() != g.deg(u)) return false;
    std::sort(s.begin(), s.end());
    if (!std::equal(s.begin(), s.end(), g.row(u))) return false;  // a duplicate shows up as a mismatch
  }
  return true;
}

// BCV1 text container (biclique.hpp:66-73): "BCV1 n", then per
// biclique "B k", a line of the k source ids, a line "t c_1 ... c_t"; then
// "R" and one "u v" line per residual edge.  Ids ascending, bicliques in
// emission order.  Loading validates the grammar (FormatError for a wrong
// header, CorruptionError for malformed or inconsistent contents).
std::string save_cover_text(const BicliqueCover& c) {
  std::ostringstream o;
  o << "BCV1 " << c.n << "\n";
  for (const Biclique& b : c.bicliques) {
    o << "B " << b.sources.size() << "\n";
    for (size_t i = 0; i < b.sources.size(); ++i) o << (i ? " " : "") << b.sources[i];
    o << "\n" << b.targets.size();
    for (uint32_t t : b.targets) o << " " << t;
    o << "\n";
  }
  o << "R\n";
  for (const auto& e : c.residual) o << e.first << " " << e.second << "\n";
  return o.str();
}

BicliqueCover load_cover_text(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line)) throw FormatError("BCV1: empty input");
  BicliqueCover c;
  {
    std::istringstream h(line);
    std::string magic;
    long long n = -1;
    if (!(h >> magic) || magic != "BCV1") throw FormatError("BCV1: bad magic");
    if (!(h >> n) || n < 0 || n > 0xffffffffll) throw CorruptionError("BCV1: corrupt header");
    std::string extra;
    if (h >> extra) throw CorruptionError("BCV1: corrupt header");
    c.n = (uint32_t)n;
  }
  auto ids = [](const std::string& l, std::vector<uint32_t>& out) {
    std::istringstream s(l);
    long long v;
    while (s >> v) {
      if (v < 0 || v > 0xffffffffll) throw CorruptionError("BCV1: corrupt id");
      out.push_back((uint32_t)v);
    }
    if (!s.eof()) throw CorruptionError("BCV1: corrupt id list");
  };
  bool residual = false;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    if (!residual && line == "R") {
      residual = true;
      continue;
    }
    if (residual) {
      std::vector<uint32_t> uv;
      ids(line, uv);
      if (uv.size() != 2) throw CorruptionError("BCV1: corrupt residual line");
      c.residual.emplace_back(uv[0], uv[1]);
      continue;
    }
    std::istringstream s(line);
    std::string tag;
    long long k = -1;
    if (!(s >> tag >> k) || tag != "B" || k < 1) throw CorruptionError("BCV1: corrupt biclique header");
    Biclique b;
    std::string l1, l2;
    if (!std::getline(in, l1) || !std::getline(in, l2)) throw CorruptionError("BCV1: truncated biclique");
    ids(l1, b.sources);
    std::vector<uint32_t> t;
    ids(l2, t);
    if ((long long)b.sources.size() != k || t.empty() || t[0] != t.size() - 1)
      throw CorruptionError("BCV1: corrupt biclique counts");
    b.targets.assign(t.begin() + 1, t.end());
    c.bicliques.push_back(std::move(b));
  }
  if (!residual) throw CorruptionError("BCV1: truncated (no residual section)");
  try {
    validate_cover_structure(c);
  } catch (const std::exception& e) {
    throw CorruptionError(std::string("BCV1: corrupt cover: ") + e.what());
  }
  return c;
}

void save_cover_file(const BicliqueCover& c, const std::string& path) {
  std::ofstream f(path, std::ios::trunc);
  if (!f) throw std::invalid_argument("BCV1: cannot open " + path + " for writing");
  f << save_cover_text(c);
  if (!f) throw std::runtime_error("BCV1: write failed: " + path);
}

BicliqueCover load_cover_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::invalid_argument("BCV1: cannot open " + path);
  std::stringstream b;
  b << f.rdbuf();
  return load_cover_text(b.str());
}

// Device layout of the product: T (bicliques x targets) and M (rows x
// [residual columns | n + r per biclique r with the row as a source]).
void build_cover_layout(const BicliqueCover& c, CoverLayout& L) {
  const uint32_t n = c.n;
  const uint64_t nb = c.bicliques.size();
  L.n = n;
  L.nb = nb;
  L.t_off.assign(nb + 1, 0);
  for (uint64_t r = 0; r < nb; ++r) L.t_off[r + 1] = L.t_off[r] + c.bicliques[r].targets.size();
  L.t_cols.resize(L.t_off[nb]);
  for (uint64_t r = 0; r < nb; ++r)
    std::copy(c.bicliques[r].targets.begin(), c.bicliques[r].targets.end(), L.t_cols.begin() + L.t_off[r]);
  std::vector<uint64_t> cnt(n + 1, 0);
  for (const auto& e : c.residual) ++cnt[e.first + 1];
  for (const Biclique& b : c.bicliques)
    for (uint32_t u : b.sources) ++cnt[u + 1];
  for (uint32_t u = 0; u < n; ++u) cnt[u + 1] += cnt[u];
  L.m_off = cnt;
  L.m_cols.resize(cnt[n]);
  std::vector<uint64_t> pos(cnt.begin(), cnt.end() - 1);
  for (const auto& e : c.residual) L.m_cols[pos[e.first]++] = e.second;  // residual sorted: ascending per row
  for (uint64_t r = 0; r < nb; ++r)
    for (uint32_t u : c.bicliques[r].sources) {
      if ((uint64_t)n + r > 0xffffffffull) throw std::invalid_argument("biclique cover: too many bicliques for u32 ids");
      L.m_cols[pos[u]++] = (uint32_t)(n + r);
    }
}

}  // namespace cmvg
