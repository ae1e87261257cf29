// Drop-in demo: code written against the reference's operator interface
// (cmv::MatvecKernel, pagerank.hpp:25-34) runs unchanged on the B200 kernel.
//
//   drop_in_pagerank <n> <out.bin>
// builds a copy-model graph, BV-encodes A^T, wraps it in cmv::BvGpuKernel, runs
// (a) a host power iteration written purely against `const MatvecKernel&`
// (the shape of the reference's cmv::pagerank, pagerank.hpp:83-102) and
// (b) the device-resident pagerank_device(); writes both rank vectors.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cmv_b200/bv_gpu_kernel.hpp"

namespace {

// A caller that only knows the reference interface.
cmv::PageRankResult host_pagerank(const cmv::MatvecKernel& at, const cmv::DegreeVector& deg,
                                  const cmv::PageRankConfig& cfg) {
  const cmv::VertexId n = at.dimension();
  std::vector<double> p(n, 1.0 / n), q(n), y(n);
  cmv::PageRankResult r;
  for (std::uint32_t t = 1; t <= cfg.iterations; ++t) {
    double dang = 0.0;
    for (cmv::VertexId j = 0; j < n; ++j) {
      q[j] = deg[j] ? p[j] / deg[j] : 0.0;
      if (!deg[j]) dang += p[j];
    }
    at.multiply(q, y);
    const double share = cfg.dangling == cmv::DanglingPolicy::kUniform ? dang / n : 0.0;
    for (cmv::VertexId i = 0; i < n; ++i) p[i] = cfg.alpha / n + (1.0 - cfg.alpha) * (y[i] + share);
    r.iterations_run = t;
  }
  r.ranks = p;
  return r;
}

void check(int rc) { cmv::cmvg_throw_if(rc); }

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s n out.bin\n", argv[0]);
    return 2;
  }
  const uint32_t n = (uint32_t)std::atoi(argv[1]);
  cmvg_csr *g = nullptr, *gt = nullptr;
  check(cmvg_gen_copy_model(n, 24.0, 0.7, 0.8, 0x170807271ull + 3, &g));
  check(cmvg_csr_transpose(g, &gt));
  cmv::DegreeVector deg(n);
  const uint64_t* ro = cmvg_csr_row_offsets(g);
  for (uint32_t u = 0; u < n; ++u) deg[u] = (uint32_t)(ro[u + 1] - ro[u]);
  cmvg_bv_params bp{7, 3, 4, 3, 1024};
  cmvg_bvstream* s = nullptr;
  check(cmvg_bv_encode(gt, &bp, &s));
  cmv::BvGpuKernel kernel(s);  // the drop-in
  cmvg_bv_free(s);
  cmv::PageRankConfig cfg;
  cfg.iterations = 30;
  const cmv::PageRankResult a = host_pagerank(kernel, deg, cfg);
  const cmv::PageRankResult b = kernel.pagerank_device(deg, cfg);
  std::FILE* f = std::fopen(argv[2], "wb");
  std::fwrite(a.ranks.data(), 8, n, f);
  std::fwrite(b.ranks.data(), 8, n, f);
  std::fclose(f);
  double sa = 0, sb = 0;
  for (uint32_t i = 0; i < n; ++i) {
    sa += a.ranks[i];
    sb += b.ranks[i];
  }
  std::printf("{\"n\": %u, \"adds_per_product\": %llu, \"sum_host_loop\": %.17g, \"sum_device\": %.17g, "
              "\"reference_api\": %d}\n",
              n, (unsigned long long)kernel.adds_per_product(), sa, sb, CMV_B200_REFERENCE_API);
  cmvg_csr_free(g);
  cmvg_csr_free(gt);
  return 0;
}
