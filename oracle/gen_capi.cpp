// TEST INFRASTRUCTURE ONLY: the seeded workload generators
// (paper_1708_07271_b200/csrc/host/gen.cpp, compiled from the same source) as
// a standalone C library, so the CPU reference arm of bench.py builds its
// input graphs without loading the product library libcmvg.so.
#include <cstdint>
#include <cstring>
#include <new>

#include "../paper_1708_07271_b200/csrc/host/host.hpp"

extern "C" {

struct gen_csr {
  cmvg::HostCsr g;
};

int gen_copy_model(uint32_t n, double mean_degree, double p_ref, double p_copy, uint64_t seed, gen_csr** out) {
  try {
    cmvg::CopyModelParams p;
    p.n = n;
    p.mean_degree = mean_degree;
    p.p_ref = p_ref;
    p.p_copy = p_copy;
    p.seed = seed;
    auto* c = new gen_csr;
    c->g = cmvg::generate_copy_model(p);
    *out = c;
    return 0;
  } catch (...) {
    return 1;
  }
}

int gen_social(uint32_t n, uint64_t seed, gen_csr** out) {
  try {
    cmvg::SocialParams p;
    p.n = n;
    p.seed = seed;
    auto* c = new gen_csr;
    c->g = cmvg::generate_social(p);
    *out = c;
    return 0;
  } catch (...) {
    return 1;
  }
}

uint32_t gen_n(const gen_csr* g) { return g->g.n; }
uint64_t gen_m(const gen_csr* g) { return g->g.m(); }
const uint64_t* gen_row_offsets(const gen_csr* g) { return g->g.row_offsets.data(); }
const uint32_t* gen_cols(const gen_csr* g) { return g->g.cols.data(); }
void gen_free(gen_csr* g) { delete g; }
}
