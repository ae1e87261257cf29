// TEST INFRASTRUCTURE ONLY: flat C entry points over the CPU oracle for the
// Python tests and bench.py's CPU legs (ctypes).  Not part of the product.
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

#include "cmv_oracle.hpp"

using namespace cmv_oracle;

namespace {
thread_local std::string g_err;
template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 8;
  }
}
CsrGraph view_csr(uint32_t n, const uint64_t* ro, const uint32_t* cols) {
  CsrGraph g;
  g.n = n;
  g.row_offsets.assign(ro, ro + (size_t)n + 1);
  g.columns.assign(cols, cols + ro[n]);
  return g;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }
unsigned oracle_hw_threads() { return std::max(1u, std::thread::hardware_concurrency()); }

// ---- CSR objects ----
void* oracle_csr_new(uint32_t n, const uint64_t* ro, const uint32_t* cols) {
  CsrGraph* g = nullptr;
  if (guard([&] { g = new CsrGraph(view_csr(n, ro, cols)); })) return nullptr;
  return g;
}
void* oracle_build_csr(const uint32_t* pairs, uint64_t m, uint32_t n) {
  CsrGraph* g = nullptr;
  int rc = guard([&] {
    std::vector<Edge> e(m);
    for (uint64_t k = 0; k < m; ++k) e[k] = {pairs[2 * k], pairs[2 * k + 1]};
    g = new CsrGraph(build_csr(std::move(e), n));
  });
  return rc ? nullptr : g;
}
void* oracle_transpose(const void* h) {
  CsrGraph* t = nullptr;
  if (guard([&] { t = new CsrGraph(transpose(*(const CsrGraph*)h)); })) return nullptr;
  return t;
}
uint32_t oracle_csr_n(const void* h) { return ((const CsrGraph*)h)->n; }
uint64_t oracle_csr_m(const void* h) { return ((const CsrGraph*)h)->num_edges(); }
const uint64_t* oracle_csr_offsets(const void* h) { return ((const CsrGraph*)h)->row_offsets.data(); }
const uint32_t* oracle_csr_cols(const void* h) { return ((const CsrGraph*)h)->columns.data(); }
void oracle_csr_free(void* h) { delete (CsrGraph*)h; }
int oracle_out_degrees(const void* h, uint32_t* out) {
  return guard([&] {
    auto d = out_degrees(*(const CsrGraph*)h);
    std::memcpy(out, d.data(), d.size() * 4);
  });
}

int oracle_matvec_csr(const void* h, const double* x, double* y, unsigned threads) {
  return guard([&] {
    const CsrGraph& g = *(const CsrGraph*)h;
    matvec_csr_into(g, std::span<const double>(x, g.n), std::span<double>(y, g.n), threads);
  });
}
// raw-array variant (no copy of the graph)
int oracle_matvec_csr_raw(uint32_t n, const uint64_t* ro, const uint32_t* cols, const double* x, double* y,
                          unsigned threads) {
  return guard([&] {
    auto body = [&](uint32_t b, uint32_t e) {
      for (uint32_t i = b; i < e; ++i) {
        double s = 0.0;
        for (uint64_t k = ro[i]; k < ro[i + 1]; ++k) s += x[cols[k]];
        y[i] = s;
      }
    };
    if (threads <= 1) return body(0, n);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
      pool.emplace_back(body, (uint32_t)((uint64_t)n * t / threads), (uint32_t)((uint64_t)n * (t + 1) / threads));
    for (auto& th : pool) th.join();
  });
}

// ---- referenced matrix ----
void* oracle_compress(const void* h, uint32_t window, unsigned threads) {
  ReferencedMatrix* rm = nullptr;
  if (guard([&] { rm = new ReferencedMatrix(compress(*(const CsrGraph*)h, window, threads)); })) return nullptr;
  return rm;
}
void oracle_rm_free(void* h) { delete (ReferencedMatrix*)h; }
int oracle_rm_validate(const void* h) { return guard([&] { validate(*(const ReferencedMatrix*)h); }); }
int oracle_rm_arrays(const void* h, const uint32_t** refs, const uint64_t** po, const uint32_t** pc, const uint64_t** mo,
                     const uint32_t** mc, uint64_t* np, uint64_t* nm) {
  const ReferencedMatrix& rm = *(const ReferencedMatrix*)h;
  *refs = rm.refs.data();
  *po = rm.plus_offsets.data();
  *pc = rm.plus_columns.data();
  *mo = rm.minus_offsets.data();
  *mc = rm.minus_columns.data();
  *np = rm.plus_columns.size();
  *nm = rm.minus_columns.size();
  return 0;
}
void* oracle_rm_new(uint32_t n, const uint32_t* refs, const uint64_t* po, const uint32_t* pc, const uint64_t* mo,
                    const uint32_t* mc) {
  auto* rm = new ReferencedMatrix;
  rm->n = n;
  rm->refs.assign(refs, refs + n);
  rm->plus_offsets.assign(po, po + (size_t)n + 1);
  rm->minus_offsets.assign(mo, mo + (size_t)n + 1);
  rm->plus_columns.assign(pc, pc + po[n]);
  rm->minus_columns.assign(mc, mc + mo[n]);
  return rm;
}
int oracle_stats(const void* rmh, const void* gh, uint64_t* out /* n,m,m',self,max_chain,by_conv */, double* ratio) {
  return guard([&] {
    CompressionStats s = stats(*(const ReferencedMatrix*)rmh, *(const CsrGraph*)gh);
    out[0] = s.n;
    out[1] = s.m;
    out[2] = s.m_prime;
    out[3] = s.rows_self_coded;
    out[4] = s.max_chain;
    out[5] = s.ratio_by_convention;
    *ratio = s.ratio;
  });
}
int oracle_reconstruct_row(const void* h, uint32_t i, uint32_t* out, uint64_t cap, uint64_t* len) {
  return guard([&] {
    auto r = reconstruct_row(*(const ReferencedMatrix*)h, i);
    *len = r.size();
    if (r.size() <= cap) std::memcpy(out, r.data(), r.size() * 4);
  });
}
void* oracle_reconstruct_graph(const void* h) {
  CsrGraph* g = nullptr;
  if (guard([&] { g = new CsrGraph(reconstruct_graph(*(const ReferencedMatrix*)h)); })) return nullptr;
  return g;
}
int oracle_matvec_ref(const void* h, const double* x, double* y, uint64_t* adds, uint64_t* refs_used) {
  return guard([&] {
    const ReferencedMatrix& rm = *(const ReferencedMatrix*)h;
    OpCount oc = matvec_ref_into(rm, std::span<const double>(x, rm.n), std::span<double>(y, rm.n));
    if (adds) *adds = oc.adds;
    if (refs_used) *refs_used = oc.references_used;
  });
}
// Throughput mode for the CPU baseline: `threads` independent products over
// the same matrix (SPEC.md:228 allows concurrent products), each writing its
// own output.  Returns wall seconds.
double oracle_matvec_ref_concurrent(const void* h, const double* x, double* ys, unsigned threads) {
  const ReferencedMatrix& rm = *(const ReferencedMatrix*)h;
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      matvec_ref_into(rm, std::span<const double>(x, rm.n), std::span<double>(ys + (size_t)t * rm.n, rm.n));
    });
  for (auto& th : pool) th.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- pagerank ----
static int run_pr(const MatvecKernel& k, const uint32_t* deg, double alpha, uint32_t iters, double tol, int dangling,
                  const double* start, double* out, uint32_t* iters_run) {
  return guard([&] {
    PageRankConfig cfg;
    cfg.alpha = alpha;
    cfg.iterations = iters;
    if (tol >= 0) cfg.l1_tolerance = tol;
    cfg.dangling = dangling ? DanglingPolicy::kDrop : DanglingPolicy::kUniform;
    uint32_t n = k.dimension();
    DegreeVector d(deg, deg + n);
    RankVector st;
    if (start) st.assign(start, start + n);
    PageRankResult r = pagerank(k, d, cfg, start ? &st : nullptr);
    std::memcpy(out, r.ranks.data(), (size_t)n * 8);
    if (iters_run) *iters_run = r.iterations_run;
  });
}
int oracle_pagerank_csr(const void* at, const uint32_t* deg, double alpha, uint32_t iters, double tol, int dangling,
                        const double* start, double* out, uint32_t* iters_run, unsigned threads) {
  CsrKernel k(*(const CsrGraph*)at, threads);
  return run_pr(k, deg, alpha, iters, tol, dangling, start, out, iters_run);
}
int oracle_pagerank_ref(const void* rm, const uint32_t* deg, double alpha, uint32_t iters, double tol, int dangling,
                        const double* start, double* out, uint32_t* iters_run) {
  RefKernel k(*(const ReferencedMatrix*)rm);
  return run_pr(k, deg, alpha, iters, tol, dangling, start, out, iters_run);
}

}  // extern "C"
