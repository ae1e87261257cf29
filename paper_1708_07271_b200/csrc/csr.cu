// Uncompressed CSR product y = A x^T on the GPU -- the comparison point for
// the compressed kernels at equal hardware (the paper's
// S = t/t' column, compares matvec_csr against the compressed
// product).  It computes the reference's `matvec_csr` (csr.hpp:48-55,
// SPEC.md:46-90): y_i = sum of x_j over row i, exactly m adds, on the
// reference's CsrGraph arrays (u64 row offsets, u32 columns).
//
// CSR-stream (one CTA of 256 threads per 256 consecutive rows): the CTA
// streams the block's column indices with coalesced evict-first loads
// (batches of 8 independent loads per thread), writes x at each column into
// a shared value list, then each thread sums its own row from the list.
// Blocks with more than kCsrCap entries take a warp per row.  fp64 sums.
// Algorithmic bytes 4m + 8(n+1) + 8n plus the x gathers.  It is a
// comparison point, not a roofline-tuned kernel: measured ~1.6 TB/s at C2
// (latency-bound on the dependent column -> x loads); bench.py reports it
// with the CSR roofline time (its bytes at peak HBM bandwidth) beside it.
#include "internal.hpp"

namespace cmvg {

constexpr uint32_t kCsrRows = 256;  // rows per CTA (= threads)
constexpr uint32_t kCsrCap = 6144;  // staged entries per CTA (48 KB of fp64)

__global__ void __launch_bounds__(kCsrRows) csr_matvec_kernel(uint32_t n, const uint64_t* __restrict__ ro,
                                                               const uint32_t* __restrict__ cols,
                                                               const double* __restrict__ x,
                                                               double* __restrict__ y) {
  extern __shared__ __align__(16) double s_v[];
  __shared__ uint64_t s_ro[kCsrRows + 1];
  const uint32_t tid = threadIdx.x, r0 = blockIdx.x * kCsrRows, nr = min(kCsrRows, n - r0);
  for (uint32_t i = tid; i <= nr; i += kCsrRows) s_ro[i] = __ldg(ro + r0 + i);
  __syncthreads();
  auto xat = [&](uint32_t c) { return __ldg(x + c); };
  const uint64_t e0 = s_ro[0], e1 = s_ro[nr];
  if (e1 - e0 <= kCsrCap) {
    const uint32_t ne = (uint32_t)(e1 - e0);
    // batches of 8 column loads issued back to back, then their x values
    for (uint32_t base = tid; base < ne; base += 8 * kCsrRows) {
      uint32_t c[8];
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) {
        const uint32_t i = base + q * kCsrRows;
        c[q] = i < ne ? __ldcs(cols + e0 + i) : 0u;
      }
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) {
        const uint32_t i = base + q * kCsrRows;
        if (i < ne) s_v[i] = xat(c[q]);
      }
    }
    __syncthreads();
    if (tid < nr) {
      double s = 0.0;
      for (uint32_t i = (uint32_t)(s_ro[tid] - e0), e = (uint32_t)(s_ro[tid + 1] - e0); i < e; ++i) s += s_v[i];
      y[r0 + tid] = s;
    }
    return;
  }
  const uint32_t lane = tid & 31u;
  for (uint32_t r = tid >> 5; r < nr; r += kCsrRows / 32) {  // long rows: a warp per row
    double s = 0.0;
    for (uint64_t k = s_ro[r] + lane; k < s_ro[r + 1]; k += 32) s += xat(__ldcs(cols + k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[r0 + r] = s;
  }
}

}  // namespace cmvg

extern "C" int cmvg_csr_matvec_f64(uint32_t n, uint64_t m, const uint64_t* row_offsets, const uint32_t* cols,
                                   const double* x, double* y, void* stream) {
  using namespace cmvg;
  return guarded([&] {
    require(row_offsets && x && y && (cols || m == 0), "null argument");
    if (n == 0) return;
    static std::atomic<bool> attr{false};  // the attribute is per function: once per process
    if (!attr.load()) {
      CUDA_TRY(cudaFuncSetAttribute(csr_matvec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCsrCap * 8));
      attr.store(true);
    }
    csr_matvec_kernel<<<(n + kCsrRows - 1) / kCsrRows, kCsrRows, kCsrCap * 8, (cudaStream_t)stream>>>(
        n, row_offsets, cols, x, y);
    CUDA_TRY(cudaGetLastError());
  });
}
