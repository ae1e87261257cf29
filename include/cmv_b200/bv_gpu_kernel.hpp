// cmv::BvGpuKernel -- the B200 drop-in for the reference's differential
// kernel (cmv::RefKernel, reference pagerank.hpp:48-61): a cmv::MatvecKernel
// computing y = A^T x on a BV-compressed A^T with the sm_100a kernels behind
// the C ABI (include/cmvg.h).  Header-only; link libcmvg.so.
//
//   multiply()          host spans: H2D, one device product, D2H (the
//                       reference-facing, synchronous path)
//   multiply_device()   device pointers on a stream (no copies)
//   pagerank_device()   the whole power iteration on the device
//
// Errors map to the reference's exception types:
// CMVG_ERR_INVALID -> std::invalid_argument, CMVG_ERR_RANGE ->
// std::out_of_range, CMVG_ERR_CORRUPT/FORMAT -> std::runtime_error subclasses
// (cmv::CorruptionError / cmv::FormatError when the reference's rmv_io.hpp is
// available), anything else -> std::runtime_error.
#pragma once
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>

#include "../cmvg.h"

#if __has_include(<cmv/pagerank.hpp>)
#include <cmv/pagerank.hpp>
#define CMV_B200_REFERENCE_API 1
#else
#include "cmv_api.hpp"
#define CMV_B200_REFERENCE_API 0
#endif
#if __has_include(<cmv/rmv_io.hpp>)
#include <cmv/rmv_io.hpp>
#define CMV_B200_REFERENCE_ERRORS 1
#else
#define CMV_B200_REFERENCE_ERRORS 0
#endif

namespace cmv {

inline void cmvg_throw_if(int rc) {
  if (rc == CMVG_OK) return;
  const std::string msg = cmvg_last_error();
  switch (rc) {
    case CMVG_ERR_INVALID:
      throw std::invalid_argument(msg);
    case CMVG_ERR_RANGE:
      throw std::out_of_range(msg);
#if CMV_B200_REFERENCE_ERRORS
    case CMVG_ERR_FORMAT:
      throw FormatError(msg);
    case CMVG_ERR_CORRUPT:
      throw CorruptionError(msg);
#endif
    default:
      throw std::runtime_error("cmvg: " + msg);
  }
}

class BvGpuKernel final : public MatvecKernel {
 public:
  // bv_of_transpose: canonical BV stream of A^T (cmvg_bv_encode of
  // transpose(g)); the stream may be freed after construction.
  explicit BvGpuKernel(const cmvg_bvstream* bv_of_transpose, const cmvg_create_opts* opts = nullptr) {
    cmvg_throw_if(cmvg_create(bv_of_transpose, opts, &g_));
  }
  BvGpuKernel(const BvGpuKernel&) = delete;
  BvGpuKernel& operator=(const BvGpuKernel&) = delete;
  BvGpuKernel(BvGpuKernel&& o) noexcept : g_(std::exchange(o.g_, nullptr)) {}
  ~BvGpuKernel() override { cmvg_destroy(g_); }

  VertexId dimension() const override { return cmvg_dimension(g_); }

  // pagerank.hpp:31-32 contract: |x| = |y| = n, x and y do not alias.
  void multiply(std::span<const double> x, std::span<double> y) const override {
    const auto n = dimension();
    if (x.size() != n || y.size() != n) throw std::invalid_argument("BvGpuKernel::multiply: dimension mismatch");
    cmvg_throw_if(cmvg_matvec_f64(g_, x.data(), y.data(), CMVG_GATHER, CMVG_HOST, nullptr));
  }

  std::uint64_t adds_per_product() const override { return cmvg_adds_per_product(g_); }

  // ---- device extensions ----------------------------------------------------
  void multiply_device(const double* x, double* y, void* stream = nullptr) const {
    cmvg_throw_if(cmvg_matvec_f64(g_, x, y, CMVG_GATHER, CMVG_DEVICE, stream));
  }
  void multiply_device_f32(const float* x, float* y, void* stream = nullptr) const {
    cmvg_throw_if(cmvg_matvec_f32(g_, x, y, CMVG_GATHER, CMVG_DEVICE, stream));
  }
  // cmv::pagerank (pagerank.hpp:100-102) with the power iteration on the
  // device; `start` as in the reference (starting and restart distribution)
  PageRankResult pagerank_device(const DegreeVector& degrees, const PageRankConfig& cfg,
                                 const RankVector* start = nullptr) const {
    if (degrees.size() != dimension()) throw std::invalid_argument("pagerank: degree vector dimension mismatch");
    if (start && start->size() != dimension()) throw std::invalid_argument("pagerank: start dimension mismatch");
    PageRankResult r;
    r.ranks.resize(dimension());
    const int pol = cfg.dangling == DanglingPolicy::kUniform ? CMVG_DANGLING_UNIFORM : CMVG_DANGLING_DROP;
    cmvg_throw_if(cmvg_pagerank_ex(g_, degrees.data(), cfg.alpha, cfg.iterations,
                                   cfg.l1_tolerance ? *cfg.l1_tolerance : -1.0, pol, start ? start->data() : nullptr,
                                   r.ranks.data(), &r.iterations_run, CMVG_HOST, nullptr));
    return r;
  }
  cmvg_graph* handle() const { return g_; }

 private:
  cmvg_graph* g_ = nullptr;
};

}  // namespace cmv
