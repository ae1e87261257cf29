// Uncompressed CSR product y = A x^T on the GPU -- the comparison point for
// the compressed kernels at equal hardware (the paper's
// S = t/t' column, compares matvec_csr against the compressed
// product).  It computes the reference's `matvec_csr` (csr.hpp:48-55,
// SPEC.md:46-90): y_i = sum of x_j over row i, exactly m adds, on the
// reference's CsrGraph arrays (u64 row offsets, u32 columns).
//
// The kernel is the CSR-stream product of cuda/csr_stream.cuh.
// Algorithmic bytes 4m + 8(n+1) + 8n plus the x gathers.  It is a
// comparison point, not a roofline-tuned kernel: measured ~1.6 TB/s at C2
// (latency-bound on the dependent column -> x loads); bench.py reports it
// with the CSR roofline time (its bytes at peak HBM bandwidth) beside it.
#include "cuda/csr_stream.cuh"
#include "internal.hpp"

extern "C" int cmvg_csr_matvec_f64(uint32_t n, uint64_t m, const uint64_t* row_offsets, const uint32_t* cols,
                                   const double* x, double* y, void* stream) {
  using namespace cmvg;
  return guarded([&] {
    if (n == 0) return;  // nothing to compute (empty vectors may have null data pointers)
    require(row_offsets && x && y && (cols || m == 0), "null argument");
    CUDA_TRY(launch_csr_stream<false>(n, row_offsets, cols, x, n, nullptr, y, (cudaStream_t)stream));
  });
}
