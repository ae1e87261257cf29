/*
 * cmvg.h -- C ABI of the B200-native compressed adjacency-matrix product.
 *
 * This is the drop-in boundary for the reference's operator surface
 * (reference proj/include/cmv/...):
 *
 *   cmvg_matvec_f64 / cmvg_matvec_f32  replace  cmv::matvec_ref_into
 *       (ref_matvec.hpp:30-31), cmv::matvec_ref (ref_matvec.hpp:34-35) and
 *       cmv::MatvecKernel::multiply (pagerank.hpp:31-32); the SCATTER form
 *       replaces cmv::matvec_ref_left (ref_matvec.hpp:40-41).
 *   cmvg_adds_per_product               replaces MatvecKernel::adds_per_product
 *       (pagerank.hpp:33).
 *   cmvg_dimension                      replaces MatvecKernel::dimension
 *       (pagerank.hpp:30).
 *   cmvg_decode_csr                     replaces cmv::reconstruct_graph
 *       (ref_matrix.hpp:75-76).
 *   cmvg_bv_encode                      replaces cmv::compress (ref_matrix.hpp:69)
 *       as the builder of the compressed form (BV stream instead of A').
 *   cmvg_pagerank                       replaces cmv::pagerank (pagerank.hpp:100-102)
 *       for a device-resident kernel.
 *   cmvg_stats / cmvg_graph_info        replace cmv::stats (ref_matrix.hpp:89).
 *
 * Conventions: opaque handles, int status codes, no
 * exceptions across the ABI; cmvg_last_error() returns a thread-local
 * message.  Status codes map to the reference's exception types:
 * CMVG_ERR_INVALID -> std::invalid_argument, CMVG_ERR_RANGE ->
 * std::out_of_range, CMVG_ERR_FORMAT -> cmv::FormatError, CMVG_ERR_CORRUPT ->
 * cmv::CorruptionError (rmv_io.hpp:13-22).  The device handle owns all
 * device memory; callers own their input/output buffers.  A handle may serve
 * concurrent products on distinct streams for DEVICE pointers; HOST-pointer
 * calls use per-handle staging buffers and are serialised internally.
 */
#ifndef CMVG_H_
#define CMVG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMVG_OK 0
#define CMVG_ERR_INVALID 1
#define CMVG_ERR_RANGE 2
#define CMVG_ERR_FORMAT 3
#define CMVG_ERR_CORRUPT 4
#define CMVG_ERR_CUDA 5
#define CMVG_ERR_NOMEM 6
#define CMVG_ERR_UNSUPPORTED 7
#define CMVG_ERR_INTERNAL 8

/* product forms */
#define CMVG_GATHER 0  /* y = A * x^T  (row i of y = sum over row i of A)     */
#define CMVG_SCATTER 1 /* y = x * A    (computed on A's own compression)      */
#define CMVG_LEFT 2    /* y = x * A    as (A^T) x on the transpose's compression,
                          the reference's matvec_ref_left (ref_matvec.hpp:37-41):
                          A^T, its references (cmv::compress's rule) and its
                          layout are built on the GPU on first use; whole-graph
                          handles only */
/* pointer kinds */
#define CMVG_HOST 0   /* host buffers: H2D/D2H inside the call              */
#define CMVG_DEVICE 1 /* device buffers on the handle's device (16-B aligned) */
/* interval evaluation (cmvg_create_opts.interval_mode) */
#define CMVG_INTERVALS_PREFIX 0 /* O(1) from a tile-local exclusive prefix of x */
#define CMVG_INTERVALS_DIRECT 1 /* summed from the shared-memory x window       */
/* PageRank dangling policy (cmv::DanglingPolicy, pagerank.hpp:16) */
#define CMVG_DANGLING_UNIFORM 0
#define CMVG_DANGLING_DROP 1

typedef struct cmvg_csr cmvg_csr;           /* host CSR graph (cmv::CsrGraph)   */
typedef struct cmvg_bvstream cmvg_bvstream; /* host canonical BV stream         */
typedef struct cmvg_graph cmvg_graph;       /* device handle (one GPU, one shard) */

typedef struct {
  uint32_t window;       /* w: reference window (<= 7 for the device layout) */
  uint32_t max_ref;      /* R: longest reference chain; 0 = unbounded       */
  uint32_t min_interval; /* Lmin                                             */
  uint32_t zeta_k;       /* residual zeta code parameter (3)                 */
  uint32_t segment_rows; /* references never cross a multiple of this       */
} cmvg_bv_params;

typedef struct {
  uint64_t stream_bits; /* S: canonical BV stream length                    */
  uint64_t rows_with_ref;
  uint64_t copied_edges;
  uint64_t interval_edges;
  uint64_t intervals;
  uint64_t residual_edges;
  uint64_t minus_edges; /* reference entries skipped by copy blocks        */
  uint32_t max_depth;
  uint32_t nsegments;
} cmvg_bv_stats;

typedef struct {
  int device;             /* CUDA device ordinal                              */
  uint32_t block_rows;    /* rows per CTA block (power of 2, multiple of the segment) */
  uint32_t lanes;         /* decode lanes (threads) per block                 */
  uint32_t window;        /* x-window entries staged per block                */
  uint32_t stream_cap_words; /* reserved (ignored): the sliced streams are read through L2 */
  uint32_t interval_mode; /* reserved (ignored): intervals always use the x-window prefix */
  uint32_t row_begin;     /* shard [row_begin, row_end); row_end 0 = n        */
  uint32_t row_end;
} cmvg_create_opts;

typedef struct {
  uint32_t n;
  uint64_t m;
  uint32_t row_begin, row_end;
  uint64_t bv_stream_bits;      /* canonical S (whole graph)               */
  uint64_t bvd_row_bits;        /* device-layout coded payload (shard)     */
  uint64_t bvd_stream_bytes;    /* incl. lane alignment and padding        */
  uint64_t bvd_lane_table_bytes;
  uint64_t bvd_block_table_bytes;
  uint32_t block_rows, lanes, window, nblocks, max_depth, interval_mode;
  uint64_t adds_per_product;
  uint64_t device_bytes;
  uint64_t bvd_codes;           /* body codes = decode-loop iterations     */
  uint32_t max_block_words, stream_cap_words;
  double window_coverage;       /* gathered columns inside the x-window    */
  /* BV-S (sliced layout of the gather / PageRank kernels) */
  uint64_t bvs_stream_bytes;
  uint32_t bvs_max_block_words, bvs_stream_cap_words, bvs_p995_block_words, bvs_pad;
  uint64_t bvs_slices, bvs_heavy_rows;
  uint64_t bvs_lane_words, bvs_lane_words_used; /* slice body words incl. / excl. lane padding */
  uint64_t bvs_lane_iters, bvs_lane_iters_used; /* slice decode lane-iterations incl. / excl. idle lanes */
  /* BV-T (target-sorted layout of the scatter form) */
  uint64_t bvt_stream_bytes, bvt_entries, bvt_far_slots, bvt_heavy_targets, bvt_slices;
  /* BV-F (flat term stream of the gather / PageRank kernels) */
  uint64_t bvf_stream_bytes, bvf_terms, bvf_pad_terms, bvf_slot_terms, bvf_esc_terms, bvf_esc_blocks;
  uint32_t bvf_max_K, bvf_min_cbits;
} cmvg_graph_info;

/* ---- errors -------------------------------------------------------------- */
const char* cmvg_last_error(void);

/* ---- host CSR graphs ------------------------------------------------------ */
int cmvg_csr_from_arrays(uint32_t n, const uint64_t* row_offsets, const uint32_t* cols, cmvg_csr** out);
int cmvg_gen_copy_model(uint32_t n, double mean_degree, double p_ref, double p_copy, uint64_t seed, cmvg_csr** out);
int cmvg_gen_social(uint32_t n, uint64_t seed, cmvg_csr** out);
int cmvg_csr_transpose(const cmvg_csr* g, cmvg_csr** out);
uint32_t cmvg_csr_n(const cmvg_csr* g);
uint64_t cmvg_csr_m(const cmvg_csr* g);
const uint64_t* cmvg_csr_row_offsets(const cmvg_csr* g);
const uint32_t* cmvg_csr_cols(const cmvg_csr* g);
void cmvg_csr_free(cmvg_csr* g);

/* ---- canonical BV stream (host) ------------------------------------------ */
int cmvg_bv_encode(const cmvg_csr* g, const cmvg_bv_params* p, cmvg_bvstream** out);
/* CBV1 container: the BV stream on disk (modelled on the reference's RMV1,
 * rmv_io.hpp:31-49: save_rmv / load_rmv / encode_rmv / decode_rmv).  Load
 * validates everything and returns CMVG_ERR_FORMAT for an unrecognised
 * container (bad magic or version, cmv::FormatError) and CMVG_ERR_CORRUPT for
 * inconsistent contents (truncation, trailing bytes, checksum, invariants, a
 * stream that does not decode to m edges; cmv::CorruptionError).  Equal
 * streams give identical bytes.  cmvg_bv_serialize sets *size and fills buf
 * when cap >= *size. */
int cmvg_bv_save(const cmvg_bvstream* s, const char* path);
int cmvg_bv_load(const char* path, cmvg_bvstream** out);
int cmvg_bv_serialize(const cmvg_bvstream* s, uint8_t* buf, uint64_t cap, uint64_t* size);
/* n, m and the encoding parameters of a stream (e.g. one just loaded). */
int cmvg_bv_describe(const cmvg_bvstream* s, uint32_t* n, uint64_t* m, cmvg_bv_params* p);
int cmvg_bv_deserialize(const uint8_t* buf, uint64_t size, cmvg_bvstream** out);
int cmvg_bv_from_words(uint32_t n, uint64_t m, const cmvg_bv_params* p, const uint32_t* words, uint64_t nbits,
                       const uint64_t* segment_bit_offsets, cmvg_bvstream** out);
int cmvg_bv_decode_host(const cmvg_bvstream* s, cmvg_csr** out);
/* Row i of the source adjacency, decoded from the stream (replaces
 * cmv::reconstruct_row, ref_matrix.hpp:71-73): *deg gets the row's length;
 * cols (room for cap entries; may be null to query the length) gets the
 * sorted columns.  CMVG_ERR_RANGE (std::out_of_range) if i >= n,
 * CMVG_ERR_INVALID if cap < the length and cols is not null. */
int cmvg_bv_reconstruct_row(const cmvg_bvstream* s, uint32_t i, uint32_t* cols, uint64_t cap, uint64_t* deg);
int cmvg_bv_get_stats(const cmvg_bvstream* s, cmvg_bv_stats* out);
const uint32_t* cmvg_bv_words(const cmvg_bvstream* s, uint64_t* nwords);
const uint64_t* cmvg_bv_segment_offsets(const cmvg_bvstream* s, uint64_t* count);
void cmvg_bv_free(cmvg_bvstream* s);

/* ---- device handle -------------------------------------------------------- */
void cmvg_default_opts(cmvg_create_opts* o);
int cmvg_create(const cmvg_bvstream* s, const cmvg_create_opts* opts, cmvg_graph** out);
int cmvg_destroy(cmvg_graph* g);
/* Host-only: build the device layout for `opts` and report its sizes
 * (no GPU needed; used for layout statistics and tests). */
int cmvg_layout_info(const cmvg_bvstream* s, const cmvg_create_opts* opts, cmvg_graph_info* out);
/* Host-only: build the device layout and copy it out (tests re-decode it on
 * the CPU).  words: u32[*nwords]; blocks: 8 x u32 per block
 * {word_offset lo, word_offset hi, nwords, wlo, nesc, 0, 0, 0}.  Free with
 * cmvg_layout_free. */
typedef struct cmvg_layout cmvg_layout;
int cmvg_layout_export(const cmvg_bvstream* s, const cmvg_create_opts* opts, cmvg_layout** out);
const uint32_t* cmvg_layout_words(const cmvg_layout* l, uint64_t* nwords);
/* BV-S words / block table (same 8-u32 block entries) */
const uint32_t* cmvg_layout_swords(const cmvg_layout* l, uint64_t* nwords);
const uint32_t* cmvg_layout_sblocks(const cmvg_layout* l, uint32_t* nblocks);
/* BV-T words / block table */
const uint32_t* cmvg_layout_twords(const cmvg_layout* l, uint64_t* nwords);
/* The BV-F layout a device handle's products read (built on the GPU by
 * cmvg_create unless CMVG_HOST_BUILD is set), copied to host memory: the
 * shard's words (block word offsets relative to its first block) and its
 * block table (8 u32 per block: BvfBlockInfo).  Null pointers query the
 * counts.  (Test / inspection entry point; no reference counterpart.) */
int cmvg_bvf_export(const cmvg_graph* g, uint32_t* words, uint64_t words_cap, uint32_t* blocks, uint64_t blocks_cap,
                    uint64_t* nwords, uint32_t* nblocks, int* device_built);
/* BV-F words / block table (8 u32 per block: BvfBlockInfo, host/layout.hpp) */
const uint32_t* cmvg_layout_fwords(const cmvg_layout* l, uint64_t* nwords);
const uint32_t* cmvg_layout_fblocks(const cmvg_layout* l, uint32_t* nblocks);
const uint32_t* cmvg_layout_tblocks(const cmvg_layout* l, uint32_t* nblocks);
const uint32_t* cmvg_layout_blocks(const cmvg_layout* l, uint32_t* nblocks);
void cmvg_layout_free(cmvg_layout* l);
int cmvg_graph_info_get(const cmvg_graph* g, cmvg_graph_info* out);
/* Columns of x (sorted, unique) that this handle's gather / PageRank step
 * reads: its blocks' x-windows plus their out-of-window columns.  A sharded
 * PageRank only needs these entries of q from the other shards (halo
 * exchange).  *count is always set; cols is filled when cap >= *count. */
int cmvg_read_set(const cmvg_graph* g, uint32_t* cols, uint64_t cap, uint64_t* count);

uint32_t cmvg_dimension(const cmvg_graph* g);
uint64_t cmvg_adds_per_product(const cmvg_graph* g);

/* y = A x^T (GATHER) or y = x A (SCATTER).  x has n entries; y has
 * row_end - row_begin entries for GATHER (the shard's rows) and n for SCATTER.
 * `stream` is a cudaStream_t (NULL = legacy default stream). */
int cmvg_matvec_f64(cmvg_graph* g, const double* x, double* y, int form, int ptr_kind, void* stream);
int cmvg_matvec_f32(cmvg_graph* g, const float* x, float* y, int form, int ptr_kind, void* stream);
/* Y = A X, X row-major n x k (fp32), Y (row_end-row_begin) x k. */
int cmvg_matmat_f32(cmvg_graph* g, const float* X, float* Y, uint32_t k, int ptr_kind, void* stream);
/* Decoded adjacency of the whole graph: row_offsets[n+1], cols[m]. */
int cmvg_decode_csr(cmvg_graph* g, uint64_t* row_offsets, uint32_t* cols, int ptr_kind, void* stream);

/* Uncompressed comparison point (replaces cmv::matvec_csr, csr.hpp:48-55, on
 * the GPU): y = A x^T from the reference's CsrGraph arrays (row_offsets[n+1]
 * u64, cols[m] u32), fp64, DEVICE pointers on the current device.  Used to
 * report the compressed product against plain CSR at equal hardware (the
 * paper's S = t/t' column). */
int cmvg_csr_matvec_f64(uint32_t n, uint64_t m, const uint64_t* row_offsets, const uint32_t* cols, const double* x,
                        double* y, void* stream);

/* Biclique covers (reference include/cmv/biclique.hpp): an
 * edge-disjoint decomposition of A's edges into bicliques (S_r, C_r) plus
 * residual edges, and its product on the GPU.
 *   cmvg_bicover_extract     replaces cmv::extract_greedy (biclique.hpp:58-61);
 *                            per_round = 1 emits the best candidate per round
 *                            (the reference's rule), 0 every still-valid one.
 *   cmvg_bicover_verify      replaces cmv::verify_cover (biclique.hpp:63-64).
 *   cmvg_bicover_save/load   replace cmv::save_cover / load_cover (BCV1 text,
 *                            biclique.hpp:66-73); load returns CMVG_ERR_FORMAT
 *                            for a wrong header, CMVG_ERR_CORRUPT otherwise.
 *   cmvg_bicover_matvec_f64  replaces cmv::matvec_biclique_into
 *                            (biclique.hpp:39-46): y = A x (n entries each).
 *   cmvg_bicover_sizes       compressed_size = sum |S_r|+|C_r| + |residual|
 *                            (biclique.hpp:33-34) = the product's adds.
 * Arrays: sources / targets of biclique r at [off[r], off[r+1]), residual as
 * (u, v) pairs; ids strictly ascending per side, residual sorted.  The device
 * operands are built on the first product, on the current device. */
typedef struct cmvg_bicover cmvg_bicover;
int cmvg_bicover_extract(const cmvg_csr* g, uint64_t min_gain, uint64_t max_rounds, uint32_t per_round,
                         cmvg_bicover** out);
int cmvg_bicover_from_arrays(uint32_t n, uint64_t nb, const uint64_t* src_off, const uint32_t* src,
                             const uint64_t* tgt_off, const uint32_t* tgt, uint64_t nres, const uint32_t* res_uv,
                             cmvg_bicover** out);
int cmvg_bicover_sizes(const cmvg_bicover* h, uint32_t* n, uint64_t* nb, uint64_t* nsrc, uint64_t* ntgt,
                       uint64_t* nres, uint64_t* compressed_size);
int cmvg_bicover_export(const cmvg_bicover* h, uint64_t* src_off, uint32_t* src, uint64_t* tgt_off, uint32_t* tgt,
                        uint32_t* res_uv);
int cmvg_bicover_verify(const cmvg_bicover* h, const cmvg_csr* g, int* ok);
int cmvg_bicover_save(const cmvg_bicover* h, const char* path);
int cmvg_bicover_load(const char* path, cmvg_bicover** out);
int cmvg_bicover_matvec_f64(cmvg_bicover* h, const double* x, double* y, int ptr_kind, void* stream);
void cmvg_bicover_free(cmvg_bicover* h);

/* PageRank (pagerank.hpp:83-102) on a handle holding A^T (the whole graph):
 * p_t = alpha/n + (1-alpha) (A^T q + [uniform] D/n), q = p/d.  degrees are
 * the out-degrees of A.  ranks receives n doubles. */
int cmvg_pagerank(cmvg_graph* g, const uint32_t* degrees, double alpha, uint32_t iterations, double l1_tolerance,
                  int dangling, double* ranks, uint32_t* iterations_run, int ptr_kind, void* stream);
/* cmvg_pagerank with a start vector (pagerank.hpp:100-102 `start`): the power
 * iteration starts from it and it is also the restart distribution,
 * p_t = alpha * start + (1 - alpha) * (A^T q + D/n).  It must be a
 * probability vector (non-negative, sum 1 within 1e-9; else
 * CMVG_ERR_INVALID).  start == NULL is the uniform 1/n.  start uses ptr_kind. */
int cmvg_pagerank_ex(cmvg_graph* g, const uint32_t* degrees, double alpha, uint32_t iterations, double l1_tolerance,
                     int dangling, const double* start, double* ranks, uint32_t* iterations_run, int ptr_kind,
                     void* stream);

/* One PageRank iteration on a shard (multi-GPU driver building block):
 * reads q (all n entries, device) and the dangling mass D of the previous
 * iterate, writes the shard's p' and q' = p'/d (device, shard-local) and
 * the shard's partial sums {sum_{d=0} p', sum |p' - p_prev|} into partial[2]
 * (device doubles).  p_prev may be NULL (then the L1 partial is 0). */
int cmvg_pagerank_step(cmvg_graph* g, const double* q, const uint32_t* degrees_shard, double alpha,
                       double dangling_mass, int dangling, const double* p_prev, double* p_next,
                       double* q_next, double* partial, void* stream);

/* cmvg_pagerank_step with the halo exchange fused into the kernel (multi-GPU
 * over NVLink peer memory): each new q'_k is also stored, at its global
 * column, into push_dst[p] for every bit p set in push_mask[k] (device
 * arrays: push_mask one byte per shard row, push_dst up to 8 device pointers
 * -- the peers' q buffers, e.g. CUDA IPC / symmetric memory).  The stores are
 * complete (system-scope fence) when the kernel completes; the caller orders
 * the peers' next step after it (e.g. the scalar all_reduce). */
int cmvg_pagerank_step_push(cmvg_graph* g, const double* q, const uint32_t* degrees_shard, double alpha,
                            double dangling_mass, int dangling, const double* p_prev, double* p_next,
                            double* q_next, double* partial, const uint8_t* push_mask, double* const* push_dst,
                            void* stream);

/* cmvg_pagerank_step / _push with the dangling mass read from DEVICE memory
 * (dangling_mass_dev[0], e.g. element 0 of the previous step's all-reduced
 * partial sums): no host round trip between iterations, so a multi-GPU driver
 * can queue step -> all_reduce -> step ... (or capture them in a CUDA graph).
 * push_mask / push_dst may be NULL (no fused push). */
int cmvg_pagerank_step_dev(cmvg_graph* g, const double* q, const uint32_t* degrees_shard, double alpha,
                           const double* dangling_mass_dev, int dangling, const double* p_prev, double* p_next,
                           double* q_next, double* partial, const uint8_t* push_mask, double* const* push_dst,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CMVG_H_ */
