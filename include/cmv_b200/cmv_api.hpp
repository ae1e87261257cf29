// Boundary types of the reference's operator API, restated for builds that do
// not have the reference headers on their include path.  When they are
// available (reference proj/include/cmv/pagerank.hpp), bv_gpu_kernel.hpp uses
// them instead, so BvGpuKernel derives from the reference's own
// cmv::MatvecKernel.  Names, signatures and semantics follow
//   types.hpp:10-22      VertexId, EdgeIndex, RankVector, DegreeVector
//   pagerank.hpp:16-34   DanglingPolicy, PageRankConfig, MatvecKernel
//   pagerank.hpp:78-81   PageRankResult
#pragma once
#include <cstdint>
#include <optional>
#include <span>
#include <vector>

namespace cmv {

using VertexId = std::uint32_t;
using EdgeIndex = std::uint64_t;
using RankVector = std::vector<double>;
using DegreeVector = std::vector<std::uint32_t>;

enum class DanglingPolicy { kUniform, kDrop };

struct PageRankConfig {
  double alpha = 0.15;
  std::uint32_t iterations = 10;
  std::optional<double> l1_tolerance;
  DanglingPolicy dangling = DanglingPolicy::kUniform;
};

// y = A^T x provider; implementations are immutable views (one kernel may
// serve concurrent products).
class MatvecKernel {
 public:
  virtual ~MatvecKernel() = default;
  virtual VertexId dimension() const = 0;
  virtual void multiply(std::span<const double> x, std::span<double> y) const = 0;
  virtual std::uint64_t adds_per_product() const = 0;
};

struct PageRankResult {
  RankVector ranks;
  std::uint32_t iterations_run = 0;
};

}  // namespace cmv
