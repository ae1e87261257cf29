// Device PageRank driver (the reference's cmv::pagerank, pagerank.hpp:83-102,
// SPEC.md:254-263; Eq. 1) on a handle holding BV(A^T):
// per iteration one fused kernel (gather y = A^T q + the PageRank update,
// q' = p'/d, per-block partials) and one deterministic reduction kernel
// (dangling mass and L1 step), all device resident.
#include "internal.hpp"

namespace cmvg {
namespace {

// p0 = 1/n (or the start vector), q0 = p0/d, partials of the dangling mass
// per block of 1024 rows
__global__ void pr_init_kernel(const uint32_t* __restrict__ deg, uint32_t n, const double* __restrict__ start,
                               double* __restrict__ p, double* __restrict__ q, double* __restrict__ partial) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double dang = 0.0;
  if (i < n) {
    const double p0 = start ? start[i] : 1.0 / (double)n;
    const uint32_t d = deg[i];
    p[i] = p0;
    q[i] = d ? p0 / (double)d : 0.0;
    if (!d) dang = p0;
  }
  __shared__ double ws[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dang += __shfl_down_sync(0xffffffffu, dang, o);
  if ((threadIdx.x & 31u) == 0) ws[threadIdx.x >> 5] = dang;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) s += ws[w];
    partial[2 * blockIdx.x] = s;
    partial[2 * blockIdx.x + 1] = 0.0;
  }
}

// sum partial[nb][2] -> out[2] (fixed order: deterministic)
__global__ void pr_reduce_kernel(const double* __restrict__ partial, uint32_t nb, double* __restrict__ out) {
  __shared__ double sa[1024], sb[1024];
  double a = 0.0, b = 0.0;
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    a += partial[2 * i];
    b += partial[2 * i + 1];
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (uint32_t s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sa[threadIdx.x] += sa[threadIdx.x + s];
      sb[threadIdx.x] += sb[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sa[0];
    out[1] = sb[0];
  }
}

void launch_pr_step(cmvg_graph* g, const double* q, PrArgs pr, double* p_next, cudaStream_t st) {
  launch_bvf<double, double, true>(g, q, q, p_next, pr, st);
}

}  // namespace

void run_pagerank(cmvg_graph* g, const uint32_t* degrees, double alpha, uint32_t iters, double l1_tol, int dangling,
                  const double* start, double* ranks, uint32_t* iters_run, int ptr_kind, cudaStream_t st) {
  const uint32_t n = g->n;
  // the iteration's vectors live in the handle (allocated once: a C3 call
  // would otherwise spend more time in cudaMalloc / cudaFree of its 2 GB than
  // in several iterations); concurrent calls on one handle are serialised
  std::lock_guard<std::mutex> lk(g->pr_mu);
  DevBuf ddeg;
  DevBuf& p0 = g->pr_buf[0];
  DevBuf& p1 = g->pr_buf[1];
  DevBuf& q0 = g->pr_buf[2];
  DevBuf& q1 = g->pr_buf[3];
  DevBuf& part = g->pr_buf[4];
  DevBuf& scal = g->pr_buf[5];
  const uint32_t* deg = degrees;
  DevBuf dstart;
  const double* p0v = start;  // restart distribution (null = uniform)
  if (ptr_kind == CMVG_HOST) {
    ddeg.upload(degrees, n);
    deg = ddeg.as<uint32_t>();
    if (start) {
      dstart.upload(start, n);
      p0v = dstart.as<double>();
    }
  }
  p0.alloc((size_t)n * 8 + 64);
  p1.alloc((size_t)n * 8 + 64);
  q0.alloc((size_t)n * 8 + 64);
  q1.alloc((size_t)n * 8 + 64);
  const uint32_t ib = (n + 1023) / 1024;
  part.alloc((size_t)std::max(ib, g->nblocks) * 16);
  scal.alloc(4 * 8);
  double* p = p0.as<double>();
  double* pn = p1.as<double>();
  double* q = q0.as<double>();
  double* qn = q1.as<double>();
  double* dm = scal.as<double>();  // [0] dangling mass, [1] l1
  pr_init_kernel<<<ib, 1024, 0, st>>>(deg, n, p0v, p, q, part.as<double>());
  CUDA_TRY(cudaGetLastError());
  pr_reduce_kernel<<<1, 1024, 0, st>>>(part.as<double>(), ib, dm);
  CUDA_TRY(cudaGetLastError());
  const bool use_tol = l1_tol >= 0.0;
  uint32_t t = 0;
  auto step = [&](double* pc, double* pnx, double* qc, double* qnx) {
    PrArgs pr{};
    pr.deg = deg;
    pr.p_prev = use_tol ? pc : nullptr;
    pr.q_next = qnx;
    pr.partial = part.as<double>();
    pr.dmass = dm;
    pr.alpha = alpha;
    pr.n = n;
    pr.uniform = dangling == CMVG_DANGLING_UNIFORM;
    pr.p0 = p0v;
    launch_pr_step(g, qc, pr, pnx, st);
    pr_reduce_kernel<<<1, 1024, 0, st>>>(part.as<double>(), g->nblocks, dm);
    CUDA_TRY(cudaGetLastError());
  };
  if (!use_tol && iters >= 4) {
    // fixed iteration count: two iterations (ping-pong) captured once as a
    // CUDA graph and replayed -- no per-kernel launch overhead for small graphs
    step(p, pn, q, qn);  // first launch outside the capture (kernel attributes)
    std::swap(p, pn);
    std::swap(q, qn);
    cudaStream_t cs = st;
    bool own = false;
    if (cs == nullptr) {  // the legacy default stream cannot be captured
      CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      own = true;
      CUDA_TRY(cudaStreamSynchronize(st));
    }
    cudaStream_t saved = st;
    st = cs;
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    step(p, pn, q, qn);
    step(pn, p, qn, q);
    CUDA_TRY(cudaStreamEndCapture(cs, &graph));
    CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
    const uint32_t pairs = (iters - 1) / 2;
    for (uint32_t k = 0; k < pairs; ++k) CUDA_TRY(cudaGraphLaunch(exec, cs));
    if ((iters - 1) % 2) {
      step(p, pn, q, qn);
      std::swap(p, pn);
      std::swap(q, qn);
    }
    CUDA_TRY(cudaGraphExecDestroy(exec));
    CUDA_TRY(cudaGraphDestroy(graph));
    st = saved;
    if (own) {
      CUDA_TRY(cudaStreamSynchronize(cs));
      CUDA_TRY(cudaStreamDestroy(cs));
    }
    if (iters_run) *iters_run = iters;
    CUDA_TRY(cudaMemcpyAsync(ranks, p, (size_t)n * 8, ptr_kind == CMVG_HOST ? cudaMemcpyDeviceToHost
                                                                              : cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return;
  }
  for (t = 1; t <= iters; ++t) {
    step(p, pn, q, qn);
    std::swap(p, pn);
    std::swap(q, qn);
    if (use_tol) {
      double l1 = 0.0;
      CUDA_TRY(cudaMemcpyAsync(&l1, dm + 1, 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      if (l1 <= l1_tol) break;
    }
  }
  if (t > iters) t = iters;
  if (iters_run) *iters_run = t;
  CUDA_TRY(cudaMemcpyAsync(ranks, p, (size_t)n * 8, ptr_kind == CMVG_HOST ? cudaMemcpyDeviceToHost
                                                                            : cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
}

void pagerank_step(cmvg_graph* g, const double* q, const uint32_t* deg, double alpha, double dmass, int dangling,
                   const double* p_prev, double* p_next, double* q_next, double* partial, cudaStream_t st,
                   const uint8_t* push_mask, double* const* push_dst, const double* dmass_dev) {
  StreamScratch scratch(g->device, (size_t)g->nblocks * 16 + 64, st);  // per launch (concurrent steps)
  PrArgs pr{};
  pr.push_mask = push_mask;
  pr.push_dst = push_dst;
  pr.deg = deg;
  pr.p_prev = p_prev;
  pr.q_next = q_next;
  pr.partial = scratch.as<double>();
  pr.dmass = dmass_dev;  // device scalar when given (no host round trip), else the host value
  pr.dmass_host = dmass;
  pr.alpha = alpha;
  pr.n = g->n;
  pr.uniform = dangling == CMVG_DANGLING_UNIFORM;
  launch_pr_step(g, q, pr, p_next, st);
  pr_reduce_kernel<<<1, 1024, 0, st>>>(scratch.as<double>(), g->nblocks, partial);
  CUDA_TRY(cudaGetLastError());
}

}  // namespace cmvg
