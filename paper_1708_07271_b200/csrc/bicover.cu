// Biclique-cover product on the GPU (reference
// matvec_biclique_into, include/cmv/biclique.hpp:39-46, SPEC.md:310-318,
// PAPER.md:281-287): y = A x on a cover of A's edges by bicliques (S_r, C_r)
// plus residual edges, in two data-parallel passes over two CSR operands
// built once per handle (host/biclique.cpp build_cover_layout):
//   1. c = T x        c_r = sum of x over C_r        (one row per biclique)
//   2. y = M [x ; c]  y_i = sum of x_j over i's residual edges
//                           + sum of c_r over the bicliques with i in S_r
// both with the CSR-stream kernel (cuda/csr_stream.cuh), so a biclique's
// target sum is computed once and reused by all its sources -- the
// "computation-friendly" saving: sum_r (|S_r| + |C_r|) + |residual| adds
// (compressed_size) instead of m.  Atomic-free and deterministic (the
// reference is sequential for determinism); all terms enter with
// a plus sign, so plain fp64 sums are accurate to ~(row length) ulps.
#include <memory>

#include "cuda/csr_stream.cuh"
#include "internal.hpp"

struct cmvg_bicover {
  cmvg::BicliqueCover c;
  // device operands (built on the first product, on the current device)
  std::mutex mu;
  int device = -1;
  cmvg::DevBuf t_off, t_cols, m_off, m_cols, cbuf, hx, hy;
};

using namespace cmvg;

namespace {

void ensure_device(cmvg_bicover* h) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (h->device == dev) return;
  if (h->device >= 0) throw std::invalid_argument("biclique cover: already resident on another device");
  CoverLayout L;
  build_cover_layout(h->c, L);
  h->t_off.upload(L.t_off.data(), L.t_off.size());
  h->t_cols.upload(L.t_cols.data(), L.t_cols.size());
  h->m_off.upload(L.m_off.data(), L.m_off.size());
  h->m_cols.upload(L.m_cols.data(), L.m_cols.size());
  h->cbuf.alloc(std::max<size_t>(8, L.nb * 8));
  h->device = dev;
}

}  // namespace

extern "C" {

int cmvg_bicover_extract(const cmvg_csr* g, uint64_t min_gain, uint64_t max_rounds, uint32_t per_round,
                         cmvg_bicover** out) {
  return guarded([&] {
    require(g && out, "null argument");
    auto h = std::make_unique<cmvg_bicover>();
    h->c = extract_greedy(g->g, min_gain, max_rounds, per_round);
    *out = h.release();
  });
}

int cmvg_bicover_from_arrays(uint32_t n, uint64_t nb, const uint64_t* src_off, const uint32_t* src,
                             const uint64_t* tgt_off, const uint32_t* tgt, uint64_t nres, const uint32_t* res_uv,
                             cmvg_bicover** out) {
  return guarded([&] {
    require(out && (nb == 0 || (src_off && tgt_off && src && tgt)) && (nres == 0 || res_uv), "null argument");
    auto h = std::make_unique<cmvg_bicover>();
    h->c.n = n;
    h->c.bicliques.resize(nb);
    for (uint64_t r = 0; r < nb; ++r) {
      require(src_off[r] <= src_off[r + 1] && tgt_off[r] <= tgt_off[r + 1], "biclique cover: offsets not monotone");
      h->c.bicliques[r].sources.assign(src + src_off[r], src + src_off[r + 1]);
      h->c.bicliques[r].targets.assign(tgt + tgt_off[r], tgt + tgt_off[r + 1]);
    }
    h->c.residual.resize(nres);
    for (uint64_t e = 0; e < nres; ++e) h->c.residual[e] = {res_uv[2 * e], res_uv[2 * e + 1]};
    validate_cover_structure(h->c);
    *out = h.release();
  });
}

int cmvg_bicover_sizes(const cmvg_bicover* h, uint32_t* n, uint64_t* nb, uint64_t* nsrc, uint64_t* ntgt,
                       uint64_t* nres, uint64_t* compressed_size) {
  return guarded([&] {
    require(h && n && nb && nsrc && ntgt && nres && compressed_size, "null argument");
    *n = h->c.n;
    *nb = h->c.bicliques.size();
    uint64_t s = 0, t = 0;
    for (const Biclique& b : h->c.bicliques) {
      s += b.sources.size();
      t += b.targets.size();
    }
    *nsrc = s;
    *ntgt = t;
    *nres = h->c.residual.size();
    *compressed_size = h->c.compressed_size();
  });
}

int cmvg_bicover_export(const cmvg_bicover* h, uint64_t* src_off, uint32_t* src, uint64_t* tgt_off, uint32_t* tgt,
                        uint32_t* res_uv) {
  return guarded([&] {
    require(h && src_off && tgt_off && (h->c.residual.empty() || res_uv), "null argument");
    uint64_t s = 0, t = 0;
    src_off[0] = tgt_off[0] = 0;
    for (size_t r = 0; r < h->c.bicliques.size(); ++r) {
      const Biclique& b = h->c.bicliques[r];
      std::copy(b.sources.begin(), b.sources.end(), src + s);
      std::copy(b.targets.begin(), b.targets.end(), tgt + t);
      s += b.sources.size();
      t += b.targets.size();
      src_off[r + 1] = s;
      tgt_off[r + 1] = t;
    }
    for (size_t e = 0; e < h->c.residual.size(); ++e) {
      res_uv[2 * e] = h->c.residual[e].first;
      res_uv[2 * e + 1] = h->c.residual[e].second;
    }
  });
}

int cmvg_bicover_verify(const cmvg_bicover* h, const cmvg_csr* g, int* ok) {
  return guarded([&] {
    require(h && g && ok, "null argument");
    *ok = verify_cover(h->c, g->g) ? 1 : 0;
  });
}

int cmvg_bicover_save(const cmvg_bicover* h, const char* path) {
  return guarded([&] {
    require(h && path, "null argument");
    save_cover_file(h->c, path);
  });
}

int cmvg_bicover_load(const char* path, cmvg_bicover** out) {
  return guarded([&] {
    require(path && out, "null argument");
    auto h = std::make_unique<cmvg_bicover>();
    h->c = load_cover_file(path);
    *out = h.release();
  });
}

int cmvg_bicover_matvec_f64(cmvg_bicover* h, const double* x, double* y, int ptr_kind, void* stream) {
  return guarded([&] {
    require(h && x && y, "null argument");
    require(ptr_kind == CMVG_HOST || ptr_kind == CMVG_DEVICE, "ptr_kind must be CMVG_HOST or CMVG_DEVICE");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h);
    const uint32_t n = h->c.n;
    const uint32_t nb = (uint32_t)h->c.bicliques.size();
    cudaStream_t st = (cudaStream_t)stream;
    const double* dx = x;
    double* dy = y;
    if (ptr_kind == CMVG_HOST) {
      h->hx.alloc((size_t)n * 8 + 8);
      h->hy.alloc((size_t)n * 8 + 8);
      CUDA_TRY(cudaMemcpyAsync(h->hx.p, x, (size_t)n * 8, cudaMemcpyHostToDevice, st));
      dx = h->hx.as<double>();
      dy = h->hy.as<double>();
    }
    double* c = h->cbuf.as<double>();
    CUDA_TRY(launch_csr_stream<false>(nb, h->t_off.as<uint64_t>(), h->t_cols.as<uint32_t>(), dx, n, nullptr, c, st));
    CUDA_TRY(launch_csr_stream<true>(n, h->m_off.as<uint64_t>(), h->m_cols.as<uint32_t>(), dx, n, c, dy, st));
    if (ptr_kind == CMVG_HOST) {
      CUDA_TRY(cudaMemcpyAsync(y, dy, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
    }
  });
}

void cmvg_bicover_free(cmvg_bicover* h) { delete h; }

}  // extern "C"
