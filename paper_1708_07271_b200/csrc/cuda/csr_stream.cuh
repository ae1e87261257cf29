// CSR-stream product kernel shared by the uncompressed comparison product
// (csr.cu) and the biclique-cover product (biclique.cu): one CTA of 256
// threads per 256 consecutive rows streams the rows' column indices with
// coalesced evict-first loads (batches of 8 independent loads per thread),
// writes the vector entry at each column into a shared value list, then each
// thread sums its own row from the list; blocks with more than kCsrCap
// entries take a warp per row.  fp64 sums.  TWO: the vector is the
// concatenation [x ; x2] (columns >= nx read x2[c - nx]), so y = M [x ; x2]
// needs no copy.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace cmvg {

constexpr uint32_t kCsrRows = 256;  // rows per CTA (= threads)
constexpr uint32_t kCsrCap = 6144;  // staged entries per CTA (48 KB of fp64)

template <bool TWO>
__global__ void __launch_bounds__(kCsrRows) csr_stream_kernel(uint32_t n, const uint64_t* __restrict__ ro,
                                                               const uint32_t* __restrict__ cols,
                                                               const double* __restrict__ x, uint32_t nx,
                                                               const double* __restrict__ x2,
                                                               double* __restrict__ y) {
  extern __shared__ __align__(16) double s_v[];
  __shared__ uint64_t s_ro[kCsrRows + 1];
  const uint32_t tid = threadIdx.x, r0 = blockIdx.x * kCsrRows, nr = min(kCsrRows, n - r0);
  for (uint32_t i = tid; i <= nr; i += kCsrRows) s_ro[i] = __ldg(ro + r0 + i);
  __syncthreads();
  auto xat = [&](uint32_t c) { return (TWO && c >= nx) ? __ldg(x2 + (c - nx)) : __ldg(x + c); };
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


// Launch on `st`; the dynamic shared-memory attribute is set once per
// instantiation and process.
template <bool TWO>
inline cudaError_t launch_csr_stream(uint32_t n, const uint64_t* ro, const uint32_t* cols, const double* x,
                                     uint32_t nx, const double* x2, double* y, cudaStream_t st) {
  static std::atomic<bool> attr{false};
  if (!attr.load()) {
    const cudaError_t e =
        cudaFuncSetAttribute(csr_stream_kernel<TWO>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCsrCap * 8);
    if (e != cudaSuccess) return e;
    attr.store(true);
  }
  if (n == 0) return cudaSuccess;
  csr_stream_kernel<TWO><<<(n + kCsrRows - 1) / kCsrRows, kCsrRows, kCsrCap * 8, st>>>(n, ro, cols, x, nx, x2, y);
  return cudaGetLastError();
}

}  // namespace cmvg
