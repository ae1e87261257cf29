// Internal (non-ABI) definitions shared by the ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/cmvg.h"
#include "cuda/bvf_gather.cuh"
#include "host/bvd_layout.hpp"
#include "host/host.hpp"

namespace cmvg {

// ---------------------------------------------------------------------------
// errors
extern thread_local std::string g_last_error;

struct AbiError : std::runtime_error {
  int code;
  AbiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                                   \
  do {                                                                                                   \
    cudaError_t e_ = (expr);                                                                             \
    if (e_ != cudaSuccess) throw AbiError(CMVG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename F>
inline int guarded(F&& f) {
  try {
    f();
    return CMVG_OK;
  } catch (const AbiError& e) {
    return set_error(e.code, e.what());
  } catch (const std::invalid_argument& e) {
    return set_error(CMVG_ERR_INVALID, e.what());
  } catch (const std::out_of_range& e) {
    return set_error(CMVG_ERR_RANGE, e.what());
  } catch (const FormatError& e) {
    return set_error(CMVG_ERR_FORMAT, e.what());
  } catch (const CorruptionError& e) {
    return set_error(CMVG_ERR_CORRUPT, e.what());
  } catch (const std::bad_alloc&) {
    return set_error(CMVG_ERR_NOMEM, "out of host memory");
  } catch (const std::runtime_error& e) {
    // stream validation failures come from the decoder as runtime_error
    std::string m = e.what();
    return set_error(m.find("corrupt") != std::string::npos || m.find("truncated") != std::string::npos ? CMVG_ERR_CORRUPT
                                                                                                   : CMVG_ERR_INTERNAL,
                     m);
  } catch (const std::exception& e) {
    return set_error(CMVG_ERR_INTERNAL, e.what());
  }
}

inline void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

// device buffer RAII
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t b) {
    if (p && bytes >= b) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (b == 0) return;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      p = nullptr;
      throw AbiError(CMVG_ERR_NOMEM, std::string("cudaMalloc(") + std::to_string(b) + "): " + cudaGetErrorString(e));
    }
    bytes = b;
  }
  void free_now() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
  template <typename T>
  void upload(const T* src, size_t count) {
    alloc(count * sizeof(T));
    if (count) CUDA_TRY(cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice));
  }
};

// Pinned (page-locked, mapped) host memory, grown on demand.
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void alloc(size_t b) {
    if (p && bytes >= b) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaHostAlloc(&p, b, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) {
      p = nullptr;
      throw AbiError(CMVG_ERR_NOMEM, std::string("cudaHostAlloc(") + std::to_string(b) + "): " + cudaGetErrorString(e));
    }
    bytes = b;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CUDA_TRY(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace cmvg

// ---------------------------------------------------------------------------
// opaque objects
using namespace cmvg;
struct cmvg_csr {
  HostCsr g;
};
struct cmvg_bvstream {
  // shared with the device handles built from it (they keep the stream for
  // lazy layouts and row decodes without copying it)
  std::shared_ptr<BvStream> sp = std::make_shared<BvStream>();
  BvStream& s = *sp;
  cmvg_bvstream() = default;
  cmvg_bvstream(const cmvg_bvstream&) = delete;
  cmvg_bvstream& operator=(const cmvg_bvstream&) = delete;
};
struct cmvg_layout {
  BvdLayout L;
};
struct cmvg_graph {
  int device = 0;
  uint32_t n = 0;
  uint64_t m = 0;
  BvParams params;
  BvdDims dims{};
  uint32_t row_begin = 0, row_end = 0, block_begin = 0, nblocks = 0;
  uint32_t stream_cap_words = 0;
  uint32_t interval_mode = CMVG_INTERVALS_PREFIX;
  uint64_t bv_bits = 0, adds = 0;
  BvdStats stats;
  uint32_t threads = 128;  // threads per CTA
  // BV-D layout (this shard): scatter, matmat
  DevBuf words, blocks;
  // BV-S layout (this shard): gather, PageRank
  DevBuf swords, sblocks;
  uint64_t heavy_items = 0;  // heavy-row work items of the whole graph (partial-sum slots per launch)
  uint64_t s_stream_bytes = 0;
  // BV-F layout (this shard): gather, PageRank
  DevBuf fwords, fblocks;
  // escape columns of the shard's BV-F blocks, flat in block order, and each
  // block's first escape (nblocks + 1): the values x[fesc[i]] are gathered by
  // one pre-pass per product (bvf_esc_gather) so the term loop streams them
  DevBuf fesc, fesc_base;
  std::vector<uint64_t> fesc_base_h;
  uint32_t decode_attr = 0;  // dynamic shared memory set on bv_decode_tiles
  DevBuf bv_sync;            // row-group index of the BV stream (built on the first decode)
  bool have_sync = false;
  uint64_t f_stream_bytes = 0;
  BvfStats fstats;
  std::atomic<unsigned> fgather_attr{0};
  std::atomic<uint32_t> fgather_res{0};  // resident CTAs of the BV-F gather (L2 prefetch distance)
  // lazily built layouts (ensure_layouts): the host stream and build options
  std::shared_ptr<const BvStream> host_stream;
  BvdOptions build_opts;
  std::atomic<bool> have_bvs{false}, have_bvt{false};
  std::mutex layout_mu;
  // BV-T layout (this shard): scatter; combine tables (whole graph)
  DevBuf twords, tblocks, tile_ptr, tile_blk, farp_ptr, farp;
  uint32_t tfar_begin = 0, tfar_end = 0;
  uint64_t t_stream_bytes = 0;
  BvtStats tstats;
  BvsStats sstats;
  // canonical BV stream (whole graph) for decode_csr
  DevBuf bv_words, bv_seg;
  uint64_t nseg = 0;
  // staging for host-pointer calls; streams/events of the pipelined gather
  DevBuf hx, hy;
  PinnedBuf px, py;  // pinned staging of pageable host x / y (the pipelined host path)
  std::vector<uint32_t> win_need;  // per block: x prefix its window needs (prefix max)
  std::vector<uint32_t> far_need;  // per block: x prefix its out-of-window columns need (prefix max)
  mutable std::vector<uint32_t> read_set;  // sorted columns of x this shard's gather reads
  mutable std::atomic<bool> have_read_set{false};  // (device-built handles: computed on first use)
  bool device_built = false;                       // BV-F built on the device (no BV-D stats)
  std::unique_ptr<cmvg_graph> left;  // A^T's handle (x A as (A^T) x, CMVG_LEFT), built on first use
  DevBuf pr_buf[6];                  // the device PageRank loop's p, p', q, q', partials, scalars (reused)
  std::mutex pr_mu;
  std::mutex left_mu;
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaEvent_t ev[32] = {};
  std::atomic<unsigned> gather_attr{0};  // kernel attributes set (bit per x type)
  std::atomic<uint32_t> gather_res[3] = {};  // resident CTAs of the gather variants (f64, f32, PageRank)
  cmvg_graph() = default;
  cmvg_graph(const cmvg_graph&) = delete;
  cmvg_graph& operator=(const cmvg_graph&) = delete;
  ~cmvg_graph() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    for (cudaStream_t s : {s_in, s_comp, s_out})
      if (s) cudaStreamDestroy(s);
  }
  std::mutex host_mu;
  uint64_t device_bytes() const {
    return words.bytes + blocks.bytes + swords.bytes + sblocks.bytes + fwords.bytes + fblocks.bytes + fesc.bytes + fesc_base.bytes + twords.bytes +
           tblocks.bytes + tile_ptr.bytes +
           tile_blk.bytes + farp_ptr.bytes + farp.bytes + bv_words.bytes + bv_seg.bytes + bv_sync.bytes +
           (left ? left->device_bytes() : 0);
  }
  BvdDev dev() const {
    BvdDev d{};
    d.words = words.as<uint32_t>();
    d.blocks = blocks.as<BvdBlockInfo>();
    d.d = dims;
    d.block_begin = block_begin;
    d.row_begin = row_begin;
    d.stream_cap_words = stream_cap_words;
    d.nlaunch = nblocks;
    return d;
  }
  BvdDev tdev() const {
    BvdDev d = dev();
    d.words = twords.as<uint32_t>();
    d.blocks = tblocks.as<BvdBlockInfo>();
    d.stream_cap_words = 0;
    return d;
  }
  BvdDev sdev() const {
    BvdDev d = dev();
    d.words = swords.as<uint32_t>();
    d.blocks = sblocks.as<BvdBlockInfo>();
    d.stream_cap_words = 0;  // BV-S is read from global memory (L2-prefetched)
    return d;
  }
};


namespace cmvg {
// Resident CTAs of a kernel on the device (occupancy x SMs): the gather's L2
// prefetch distance.  Computed once per handle (after the dynamic
// shared-memory attribute is set); CMVG_PREFETCH_AHEAD overrides (0 = off).
template <class K>
inline uint32_t resident_ctas(K kern, int threads, size_t smem, int device, std::atomic<uint32_t>& cache) {
  uint32_t c = cache.load();
  if (!c) {
    int occ = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess) occ = 1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) sms = 1;
    c = (uint32_t)(occ > 0 ? occ : 1) * (uint32_t)(sms > 0 ? sms : 1);
    if (const char* e = std::getenv("CMVG_PREFETCH_AHEAD")) c = (uint32_t)std::strtoul(e, nullptr, 10) | 0x80000000u;
    cache.store(c | 0x80000000u);
  }
  return c & 0x7fffffffu;
}

// Keep freed blocks in a device's default memory pool (no OS round trip per
// stream-ordered allocation); once per device.
inline void keep_pool(int device) {
  static std::atomic<uint64_t> done{0};
  const uint64_t bit = 1ull << (device & 63);
  if (done.fetch_or(bit) & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    (void)cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}

// Stream-ordered scratch for one launch (cudaMallocAsync from the device's
// pool, freed on the same stream after the launch): each launch has its own
// memory, so concurrent products on distinct streams of one handle never share
// it (cmvg.h: a handle serves concurrent DEVICE-pointer products), and a
// captured CUDA graph gets memory nodes.
struct StreamScratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  StreamScratch(int device, size_t bytes, cudaStream_t s) : st(s) {
    if (!bytes) return;
    keep_pool(device);
    CUDA_TRY(cudaMallocAsync(&p, bytes, st));
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  ~StreamScratch() {
    if (p) (void)cudaFreeAsync(p, st);
  }
  StreamScratch(const StreamScratch&) = delete;
  StreamScratch& operator=(const StreamScratch&) = delete;
};

void ensure_layouts(cmvg_graph* g, bool sliced, bool target);

// kernel entry points implemented in the other translation units
// device build of the BV-F layout (bvf_build.cu) and the device BV decoder
// (cmvg_abi.cu)
struct DeviceBuildStats {
  uint64_t adds = 0;
  uint32_t depth = 0;
  double window_coverage = 1.0;
};
bool decode_tiles_ok(const cmvg_graph* g);
void decode_device(cmvg_graph* g, uint64_t* ro, uint32_t* co, uint8_t* ref_out, cudaStream_t st);
bool device_build_bvf(cmvg_graph* g, cudaStream_t st, DeviceBuildStats& ds);
struct BvfRowsView;
bool build_bvf_from_rows(cmvg_graph* g, const BvfRowsView& view, cudaStream_t st, DeviceBuildStats& ds);
std::unique_ptr<cmvg_graph> build_left_handle(cmvg_graph* g, cudaStream_t st);
void ensure_read_set(const cmvg_graph* g);

template <typename XT, typename YT, bool PR>
void launch_bvf(cmvg_graph* g, const XT* x, const XT* xfar, YT* y, const PrArgs& pr, cudaStream_t st, uint32_t b0 = 0,
                uint32_t b1 = 0xffffffffu);
template <typename T>
void launch_scatter(cmvg_graph* g, const T* x, T* y, cudaStream_t st);
void launch_matmat(cmvg_graph* g, const float* X, float* Y, uint32_t k, cudaStream_t st);
void run_pagerank(cmvg_graph* g, const uint32_t* degrees, double alpha, uint32_t iters, double l1_tol, int dangling,
                  const double* start, double* ranks, uint32_t* iters_run, int ptr_kind, cudaStream_t st);
void pagerank_step(cmvg_graph* g, const double* q, const uint32_t* deg, double alpha, double dmass, int dangling,
                   const double* p_prev, double* p_next, double* q_next, double* partial, cudaStream_t st,
                   const uint8_t* push_mask = nullptr, double* const* push_dst = nullptr,
                   const double* dmass_dev = nullptr);
}  // namespace cmvg
