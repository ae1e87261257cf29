// TEST INFRASTRUCTURE ONLY (see cmv_oracle.hpp).  CPU restatement of the
// reference's contracts; every function cites the header line and SPEC.md
// clause it follows.
#include "cmv_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <thread>

namespace cmv_oracle {
namespace {

template <typename F>
void par_rows(VertexId n, unsigned threads, F&& f) {
  if (threads <= 1 || n < 4096) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) {
    VertexId b = (VertexId)((uint64_t)n * t / threads), e = (VertexId)((uint64_t)n * (t + 1) / threads);
    pool.emplace_back([&, b, e] { f(b, e); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

// csr.hpp:38-41: sort, dedup, keep self-loops; out_of_range
// naming the offending pair.
CsrGraph build_csr(std::vector<Edge> edges, VertexId n) {
  for (const Edge& e : edges)
    if (e.first >= n || e.second >= n)
      throw std::out_of_range("edge (" + std::to_string(e.first) + "," + std::to_string(e.second) +
                              ") has an endpoint >= n=" + std::to_string(n));
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  CsrGraph g;
  g.n = n;
  g.row_offsets.assign((size_t)n + 1, 0);
  g.columns.reserve(edges.size());
  for (const Edge& e : edges) {
    g.row_offsets[e.first + 1]++;
    g.columns.push_back(e.second);
  }
  for (VertexId u = 0; u < n; ++u) g.row_offsets[u + 1] += g.row_offsets[u];
  return g;
}

// csr.hpp:43-44.  Counting sort by column; scanning sources in
// increasing order keeps every transposed row sorted.
CsrGraph transpose(const CsrGraph& g) {
  CsrGraph t;
  t.n = g.n;
  t.row_offsets.assign((size_t)g.n + 1, 0);
  for (VertexId c : g.columns) t.row_offsets[c + 1]++;
  for (VertexId v = 0; v < g.n; ++v) t.row_offsets[v + 1] += t.row_offsets[v];
  t.columns.resize(g.columns.size());
  std::vector<EdgeIndex> cur(t.row_offsets.begin(), t.row_offsets.end() - 1);
  for (VertexId u = 0; u < g.n; ++u)
    for (EdgeIndex e = g.row_offsets[u]; e < g.row_offsets[u + 1]; ++e) t.columns[cur[g.columns[e]]++] = u;
  return t;
}

// csr.hpp:46
DegreeVector out_degrees(const CsrGraph& g) {
  DegreeVector d(g.n);
  for (VertexId u = 0; u < g.n; ++u) d[u] = g.out_degree(u);
  return d;
}

// csr.hpp:48-55: y[i] = sum over row i in column order;
// rows may be partitioned across workers (bitwise partition-independent).
void matvec_csr_into(const CsrGraph& g, std::span<const double> x, std::span<double> y, unsigned threads) {
  if (x.size() != g.n || y.size() != g.n) throw std::invalid_argument("matvec_csr: dimension mismatch");
  if (x.data() == y.data() && g.n) throw std::invalid_argument("matvec_csr_into: x and y alias");
  par_rows(g.n, threads, [&](VertexId b, VertexId e) {
    for (VertexId i = b; i < e; ++i) {
      double s = 0.0;
      for (EdgeIndex k = g.row_offsets[i]; k < g.row_offsets[i + 1]; ++k) s += x[g.columns[k]];
      y[i] = s;
    }
  });
}

RankVector matvec_csr(const CsrGraph& g, const RankVector& x, unsigned threads) {
  if (x.size() != g.n) throw std::invalid_argument("matvec_csr: dimension mismatch");
  RankVector y(g.n);
  matvec_csr_into(g, x, y, threads);
  return y;
}

// ref_matrix.hpp:13-25,54-56: structural invariants, first violation throws.
void validate(const ReferencedMatrix& rm) {
  if (rm.refs.size() != rm.n || rm.plus_offsets.size() != (size_t)rm.n + 1 || rm.minus_offsets.size() != (size_t)rm.n + 1)
    throw std::invalid_argument("ReferencedMatrix: array sizes do not match n");
  if (rm.plus_offsets[0] != 0 || rm.minus_offsets[0] != 0 || rm.plus_offsets[rm.n] != rm.plus_columns.size() ||
      rm.minus_offsets[rm.n] != rm.minus_columns.size())
    throw std::invalid_argument("ReferencedMatrix: offsets do not span the column arrays");
  for (VertexId i = 0; i < rm.n; ++i) {
    if (rm.refs[i] != kNoRef && rm.refs[i] >= i)
      throw std::invalid_argument("ReferencedMatrix: refs[" + std::to_string(i) + "] is not < i");
    if (rm.plus_offsets[i] > rm.plus_offsets[i + 1] || rm.minus_offsets[i] > rm.minus_offsets[i + 1])
      throw std::invalid_argument("ReferencedMatrix: offsets decrease");
    auto p = rm.plus_row(i), m = rm.minus_row(i);
    if (rm.refs[i] == kNoRef && !m.empty()) throw std::invalid_argument("ReferencedMatrix: self-coded row with minus entries");
    for (size_t k = 0; k < p.size(); ++k)
      if (p[k] >= rm.n || (k && p[k] <= p[k - 1])) throw std::invalid_argument("ReferencedMatrix: plus row not strict/in range");
    for (size_t k = 0; k < m.size(); ++k)
      if (m[k] >= rm.n || (k && m[k] <= m[k - 1])) throw std::invalid_argument("ReferencedMatrix: minus row not strict/in range");
    size_t a = 0, b = 0;
    while (a < p.size() && b < m.size()) {
      if (p[a] == m[b]) throw std::invalid_argument("ReferencedMatrix: plus and minus intersect");
      if (p[a] < m[b]) ++a;
      else ++b;
    }
  }
}

// ref_matrix.hpp:58-69: candidates [max(0,i-W), i),
// minimise |symmetric difference|, ties -> largest index, keep the row unless
// strictly smaller; no chain limit.
ReferencedMatrix compress(const CsrGraph& g, VertexId window, unsigned threads) {
  if (window < 1) throw std::invalid_argument("compress: window must be >= 1");
  const VertexId n = g.n;
  std::vector<VertexId> refs(n, kNoRef);
  par_rows(n, threads, [&](VertexId b, VertexId e) {
    for (VertexId i = b; i < e; ++i) {
      auto Li = g.row(i);
      uint64_t best = Li.size();
      VertexId best_c = kNoRef;
      VertexId lo = i >= window ? i - window : 0;
      for (VertexId c = i; c-- > lo;) {  // nearest first: a later tie never wins
        auto Lc = g.row(c);
        size_t a = 0, k = 0, common = 0;
        while (a < Li.size() && k < Lc.size()) {
          if (Li[a] == Lc[k]) { ++common; ++a; ++k; }
          else if (Li[a] < Lc[k]) ++a;
          else ++k;
        }
        uint64_t diff = Li.size() + Lc.size() - 2 * common;
        if (diff < best) { best = diff; best_c = c; }
      }
      refs[i] = best_c;
    }
  });
  ReferencedMatrix rm;
  rm.n = n;
  rm.refs = refs;
  rm.plus_offsets.assign((size_t)n + 1, 0);
  rm.minus_offsets.assign((size_t)n + 1, 0);
  for (VertexId i = 0; i < n; ++i) {
    auto Li = g.row(i);
    if (refs[i] == kNoRef) {
      rm.plus_columns.insert(rm.plus_columns.end(), Li.begin(), Li.end());
    } else {
      auto Lr = g.row(refs[i]);
      std::set_difference(Li.begin(), Li.end(), Lr.begin(), Lr.end(), std::back_inserter(rm.plus_columns));
      std::set_difference(Lr.begin(), Lr.end(), Li.begin(), Li.end(), std::back_inserter(rm.minus_columns));
    }
    rm.plus_offsets[i + 1] = rm.plus_columns.size();
    rm.minus_offsets[i + 1] = rm.minus_columns.size();
  }
  return rm;
}

// ref_matrix.hpp:71-73: unwind the chain.
std::vector<VertexId> reconstruct_row(const ReferencedMatrix& rm, VertexId i) {
  if (i >= rm.n) throw std::out_of_range("reconstruct_row: row " + std::to_string(i) + " >= n");
  std::vector<VertexId> chain;
  for (VertexId j = i; j != kNoRef; j = rm.refs[j]) chain.push_back(j);
  std::vector<VertexId> row, tmp;
  for (size_t k = chain.size(); k-- > 0;) {
    VertexId j = chain[k];
    auto p = rm.plus_row(j), m = rm.minus_row(j);
    tmp.clear();
    std::set_union(row.begin(), row.end(), p.begin(), p.end(), std::back_inserter(tmp));
    row.clear();
    std::set_difference(tmp.begin(), tmp.end(), m.begin(), m.end(), std::back_inserter(row));
  }
  return row;
}

// ref_matrix.hpp:75-76: one forward pass.
CsrGraph reconstruct_graph(const ReferencedMatrix& rm) {
  CsrGraph g;
  g.n = rm.n;
  g.row_offsets.assign((size_t)rm.n + 1, 0);
  std::vector<VertexId> tmp, row;
  for (VertexId i = 0; i < rm.n; ++i) {
    tmp.clear();
    row.clear();
    auto p = rm.plus_row(i), m = rm.minus_row(i);
    if (rm.refs[i] != kNoRef) {
      auto r = g.row(rm.refs[i]);
      std::set_union(r.begin(), r.end(), p.begin(), p.end(), std::back_inserter(tmp));
    } else {
      tmp.assign(p.begin(), p.end());
    }
    std::set_difference(tmp.begin(), tmp.end(), m.begin(), m.end(), std::back_inserter(row));
    g.columns.insert(g.columns.end(), row.begin(), row.end());
    g.row_offsets[i + 1] = g.columns.size();
  }
  return g;
}

// ref_matrix.hpp:78-89
CompressionStats stats(const ReferencedMatrix& rm, const CsrGraph& g) {
  CompressionStats s;
  s.n = rm.n;
  s.m = g.num_edges();
  s.m_prime = rm.m_prime();
  if (s.m_prime == 0) {
    s.ratio = 1.0;
    s.ratio_by_convention = true;
  } else {
    s.ratio = (double)s.m / (double)s.m_prime;
  }
  std::vector<VertexId> depth(rm.n, 0);
  for (VertexId i = 0; i < rm.n; ++i) {
    if (rm.refs[i] == kNoRef) s.rows_self_coded++;
    else depth[i] = depth[rm.refs[i]] + 1;
    s.max_chain = std::max(s.max_chain, depth[i]);
  }
  return s;
}

// ref_matvec.hpp:20-31: rows in increasing order; plus
// ascending then minus ascending into one scalar, then + y[refs[i]].
OpCount matvec_ref_into(const ReferencedMatrix& rm, std::span<const double> x, std::span<double> y) {
  if (x.size() != rm.n || y.size() != rm.n) throw std::invalid_argument("matvec_ref: dimension mismatch");
  OpCount oc;
  for (VertexId i = 0; i < rm.n; ++i) {
    double s = 0.0;
    for (VertexId j : rm.plus_row(i)) s += x[j];
    for (VertexId j : rm.minus_row(i)) s -= x[j];
    if (rm.refs[i] != kNoRef) {
      s += y[rm.refs[i]];
      oc.references_used++;
    }
    y[i] = s;
  }
  oc.adds = rm.m_prime() + oc.references_used;
  return oc;
}

std::pair<RankVector, OpCount> matvec_ref(const ReferencedMatrix& rm, const RankVector& x) {
  if (x.size() != rm.n) throw std::invalid_argument("matvec_ref: dimension mismatch");
  RankVector y(rm.n);
  OpCount oc = matvec_ref_into(rm, x, y);
  return {std::move(y), oc};
}

// ref_matvec.hpp:37-41: x*A as A^T x on compress(transpose(g)).
std::pair<RankVector, OpCount> matvec_ref_left(const ReferencedMatrix& rm_of_transpose, const RankVector& x) {
  return matvec_ref(rm_of_transpose, x);
}

void CsrKernel::multiply(std::span<const double> x, std::span<double> y) const { matvec_csr_into(*g_, x, y, threads_); }

RefKernel::RefKernel(const ReferencedMatrix& rm) : rm_(&rm), references_used_(0) {
  for (VertexId r : rm.refs)
    if (r != kNoRef) ++references_used_;
}
void RefKernel::multiply(std::span<const double> x, std::span<double> y) const { matvec_ref_into(*rm_, x, y); }

// pagerank.hpp:83-102, SPEC.md:254-263,282-285 (Eq. 1):
// p_t = alpha*p0 + (1-alpha)*(A^T q + [uniform] D/n), q[j] = p[j]/d[j] or 0.
PageRankResult pagerank(const MatvecKernel& at, const DegreeVector& degrees, const PageRankConfig& cfg,
                        const RankVector* start) {
  if (!(cfg.alpha > 0.0 && cfg.alpha < 1.0)) throw std::invalid_argument("pagerank: alpha must be in (0,1)");
  if (cfg.iterations == 0) throw std::invalid_argument("pagerank: iterations must be > 0");
  const VertexId n = at.dimension();
  if (n == 0) throw std::invalid_argument("pagerank: empty graph");
  if (degrees.size() != n) throw std::invalid_argument("pagerank: degree vector dimension mismatch");
  RankVector p0(n, 1.0 / n);
  if (start) {
    if (start->size() != n) throw std::invalid_argument("pagerank: start dimension mismatch");
    double s = 0.0;
    for (double v : *start) {
      if (!(v >= 0.0)) throw std::invalid_argument("pagerank: start has a negative entry");
      s += v;
    }
    if (std::fabs(s - 1.0) > 1e-9) throw std::invalid_argument("pagerank: start is not a probability vector");
    p0 = *start;
  }
  RankVector p = p0, q(n), y(n), next(n);
  PageRankResult res;
  for (uint32_t t = 1; t <= cfg.iterations; ++t) {
    double dangling = 0.0;
    for (VertexId j = 0; j < n; ++j) {
      if (degrees[j] > 0) q[j] = p[j] / degrees[j];
      else {
        q[j] = 0.0;
        dangling += p[j];
      }
    }
    at.multiply(q, y);
    const double share = cfg.dangling == DanglingPolicy::kUniform ? dangling / n : 0.0;
    double l1 = 0.0;
    for (VertexId i = 0; i < n; ++i) {
      next[i] = cfg.alpha * p0[i] + (1.0 - cfg.alpha) * (y[i] + share);
      l1 += std::fabs(next[i] - p[i]);
    }
    std::swap(p, next);
    res.iterations_run = t;
    if (cfg.l1_tolerance && l1 <= *cfg.l1_tolerance) break;
  }
  res.ranks = std::move(p);
  return res;
}

}  // namespace cmv_oracle
