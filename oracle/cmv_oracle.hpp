// TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it; the product
// (paper_1708_07271_b200) never links or calls it.
//
// A restatement of the reference's declared-but-unimplemented C++ API
// (/root/reference/proj/include/cmv/*.hpp, behaviour from SPEC.md): the
// reference ships headers only, so there is no reference binary
// to compile; these bodies follow the header contracts line by line.  Parity
// pins: every SPEC.md example for these operations is a test in
// tests/test_oracle.py (golden vectors in tests/golden/spec_examples.json).
//
// Types mirror include/cmv/types.hpp:10-22 (VertexId u32, EdgeIndex u64,
// RankVector vector<double>, DegreeVector vector<u32>).
#pragma once
#include <cstdint>
#include <optional>
#include <span>
#include <utility>
#include <vector>

namespace cmv_oracle {

using VertexId = std::uint32_t;
using EdgeIndex = std::uint64_t;
using Edge = std::pair<VertexId, VertexId>;
using RankVector = std::vector<double>;
using DegreeVector = std::vector<std::uint32_t>;

inline constexpr VertexId kNoRef = static_cast<VertexId>(-1);  // ref_matrix.hpp:11

struct CsrGraph {  // csr.hpp:16-36
  VertexId n = 0;
  std::vector<EdgeIndex> row_offsets{0};
  std::vector<VertexId> columns;
  EdgeIndex num_edges() const { return columns.size(); }
  std::span<const VertexId> row(VertexId u) const {
    return {columns.data() + row_offsets[u], columns.data() + row_offsets[u + 1]};
  }
  VertexId out_degree(VertexId u) const { return (VertexId)(row_offsets[u + 1] - row_offsets[u]); }
};

CsrGraph build_csr(std::vector<Edge> edges, VertexId n);                       // csr.hpp:41
CsrGraph transpose(const CsrGraph& g);                                         // csr.hpp:44
DegreeVector out_degrees(const CsrGraph& g);                                   // csr.hpp:46
RankVector matvec_csr(const CsrGraph& g, const RankVector& x, unsigned threads = 1);  // csr.hpp:51
void matvec_csr_into(const CsrGraph& g, std::span<const double> x, std::span<double> y,
                     unsigned threads = 1);                                    // csr.hpp:54-55

struct ReferencedMatrix {  // ref_matrix.hpp:28-52
  VertexId n = 0;
  std::vector<VertexId> refs;
  std::vector<EdgeIndex> plus_offsets{0};
  std::vector<VertexId> plus_columns;
  std::vector<EdgeIndex> minus_offsets{0};
  std::vector<VertexId> minus_columns;
  EdgeIndex m_prime() const { return plus_columns.size() + minus_columns.size(); }
  std::span<const VertexId> plus_row(VertexId i) const {
    return {plus_columns.data() + plus_offsets[i], plus_columns.data() + plus_offsets[i + 1]};
  }
  std::span<const VertexId> minus_row(VertexId i) const {
    return {minus_columns.data() + minus_offsets[i], minus_columns.data() + minus_offsets[i + 1]};
  }
};

void validate(const ReferencedMatrix& rm);                                     // ref_matrix.hpp:56
ReferencedMatrix compress(const CsrGraph& g, VertexId window, unsigned threads = 1);  // ref_matrix.hpp:69
std::vector<VertexId> reconstruct_row(const ReferencedMatrix& rm, VertexId i);  // ref_matrix.hpp:73
CsrGraph reconstruct_graph(const ReferencedMatrix& rm);                        // ref_matrix.hpp:76

struct CompressionStats {  // ref_matrix.hpp:78-86
  VertexId n = 0;
  EdgeIndex m = 0;
  EdgeIndex m_prime = 0;
  double ratio = 1.0;
  bool ratio_by_convention = false;
  VertexId rows_self_coded = 0;
  VertexId max_chain = 0;
};
CompressionStats stats(const ReferencedMatrix& rm, const CsrGraph& g);         // ref_matrix.hpp:89

struct OpCount {  // ref_matvec.hpp:13-18
  std::uint64_t adds = 0;
  std::uint64_t references_used = 0;
};
OpCount matvec_ref_into(const ReferencedMatrix& rm, std::span<const double> x, std::span<double> y);  // :30-31
std::pair<RankVector, OpCount> matvec_ref(const ReferencedMatrix& rm, const RankVector& x);          // :34-35
std::pair<RankVector, OpCount> matvec_ref_left(const ReferencedMatrix& rm_of_transpose,
                                               const RankVector& x);                                 // :40-41

enum class DanglingPolicy { kUniform, kDrop };  // pagerank.hpp:16
struct PageRankConfig {                        // pagerank.hpp:18-23
  double alpha = 0.15;
  std::uint32_t iterations = 10;
  std::optional<double> l1_tolerance;
  DanglingPolicy dangling = DanglingPolicy::kUniform;
};

class MatvecKernel {  // pagerank.hpp:27-34
 public:
  virtual ~MatvecKernel() = default;
  virtual VertexId dimension() const = 0;
  virtual void multiply(std::span<const double> x, std::span<double> y) const = 0;
  virtual std::uint64_t adds_per_product() const = 0;
};

class CsrKernel final : public MatvecKernel {  // pagerank.hpp:36-46
 public:
  explicit CsrKernel(const CsrGraph& transposed, unsigned threads = 1) : g_(&transposed), threads_(threads) {}
  VertexId dimension() const override { return g_->n; }
  void multiply(std::span<const double> x, std::span<double> y) const override;
  std::uint64_t adds_per_product() const override { return g_->num_edges(); }

 private:
  const CsrGraph* g_;
  unsigned threads_;
};

class RefKernel final : public MatvecKernel {  // pagerank.hpp:48-61
 public:
  explicit RefKernel(const ReferencedMatrix& rm_of_transpose);
  VertexId dimension() const override { return rm_->n; }
  void multiply(std::span<const double> x, std::span<double> y) const override;
  std::uint64_t adds_per_product() const override { return rm_->m_prime() + references_used_; }

 private:
  const ReferencedMatrix* rm_;
  std::uint64_t references_used_;
};

struct PageRankResult {  // pagerank.hpp:78-81
  RankVector ranks;
  std::uint32_t iterations_run = 0;
};

PageRankResult pagerank(const MatvecKernel& at, const DegreeVector& degrees, const PageRankConfig& cfg,
                        const RankVector* start = nullptr);  // pagerank.hpp:100-102

}  // namespace cmv_oracle
