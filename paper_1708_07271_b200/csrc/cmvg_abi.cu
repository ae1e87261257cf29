// C ABI (include/cmvg.h): host objects, device handle, kernel dispatch.
#include "cuda/bv_decode.cuh"
#include "internal.hpp"

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace cmvg {
thread_local std::string g_last_error;
}

// ---------------------------------------------------------------------------
namespace cmvg {
// The columns of x a shard's gather reads: its blocks' x-windows, far slots
// and escape columns (device-built handles: from the BV-F stream, on first use)
void ensure_read_set(const cmvg_graph* g) {
  if (g->have_read_set) return;
  std::lock_guard<std::mutex> lk(const_cast<cmvg_graph*>(g)->layout_mu);
  if (g->have_read_set) return;
  DeviceGuard dg(g->device);
  std::vector<BvfBlockInfo> bl(g->nblocks);
  std::vector<uint32_t> w(g->f_stream_bytes / 4);
  CUDA_TRY(cudaMemcpy(bl.data(), g->fblocks.p, bl.size() * sizeof(BvfBlockInfo), cudaMemcpyDeviceToHost));
  if (!w.empty()) CUDA_TRY(cudaMemcpy(w.data(), g->fwords.p, w.size() * 4, cudaMemcpyDeviceToHost));
  std::vector<uint64_t> bm(((uint64_t)g->n + 63) / 64, 0);
  auto mark = [&](uint64_t c) { bm[c >> 6] |= 1ull << (c & 63); };
  for (const BvfBlockInfo& b : bl) {
    const uint64_t w1 = std::min<uint64_t>(g->n, (uint64_t)b.wlo + g->dims.window);
    for (uint64_t c = b.wlo; c < w1; ++c) mark(c);
    const uint32_t* s = w.data() + b.word_offset;
    for (uint32_t q = 0; q < b.nslot; ++q) mark(s[bvf_far_off(b.nact) + q]);
    if (b.flags & kBvfFlagEsc) {
      const uint32_t* es = s + b.esc_off;
      const uint32_t* ec = es + bvf_align4(b.nact + 1u);
      for (uint32_t q = 0; q < es[b.nact]; ++q) mark(ec[q]);
    }
  }
  std::vector<uint32_t>& rs = g->read_set;
  rs.clear();
  for (uint64_t wi = 0; wi < bm.size(); ++wi)
    for (uint64_t v = bm[wi]; v; v &= v - 1) rs.push_back((uint32_t)(wi * 64 + __builtin_ctzll(v)));
  g->have_read_set = true;
}
}  // namespace cmvg

namespace cmvg {
bool decode_tiles_ok(const cmvg_graph* g) {
  return kDecTileRows % g->params.segment_rows == 0 && kDecTileRows % kDecGroup == 0 && !getenv("CMVG_SERIAL_DECODE");
}

// BV stream (device copy) -> CSR in device memory (+ each row's reference
// distance when ref_out is given; the tile decoder only).  Throws on a
// corrupt stream.
void decode_device(cmvg_graph* g, uint64_t* ro, uint32_t* co, uint8_t* ref_out, cudaStream_t st) {
  BvDev s{};
  s.words = g->bv_words.as<uint32_t>();
  s.seg_bits = g->bv_seg.as<uint64_t>();
  s.n = g->n;
  s.seg_rows = g->params.segment_rows;
  s.nseg = (uint32_t)g->nseg;
  s.window = g->params.window;
  s.min_interval = g->params.min_interval;
  s.zeta_k = g->params.zeta_k;
  StreamScratch deg(g->device, (size_t)g->n * 4, st), err(g->device, 16, st);
  CUDA_TRY(cudaMemsetAsync(err.p, 0, 4, st));
  int herr = 0;
  const int tpb = 64;
  if (!decode_tiles_ok(g)) {
    if (ref_out) throw std::logic_error("reference distances need the tile decoder");
    // serial decoder (segments that do not tile; tests): per-segment parse
    // and scan, then one thread per segment writes its rows
    StreamScratch rbit(g->device, (size_t)g->n * 8, st), segsum(g->device, g->nseg * 8, st),
        segbase(g->device, g->nseg * 8, st);
    bv_index_rows<<<(unsigned)((g->nseg + tpb - 1) / tpb), tpb, 0, st>>>(s, deg.as<uint32_t>(), rbit.as<uint64_t>(),
                                                                        segsum.as<uint64_t>(), err.as<int>());
    CUDA_TRY(cudaGetLastError());
    bv_scan_segments<<<1, 1024, 0, st>>>(segsum.as<uint64_t>(), g->nseg, 1, g->m, segbase.as<uint64_t>(),
                                         err.as<int>());
    CUDA_TRY(cudaGetLastError());
    bv_seg_decode<<<(unsigned)((g->nseg + tpb - 1) / tpb), tpb, 0, st>>>(s, segbase.as<uint64_t>(), ro, co,
                                                                        err.as<int>());
  } else {
    const uint32_t ng = (uint32_t)(((uint64_t)g->n + kDecGroup - 1) / kDecGroup);
    {  // the handle's row-group index: one serial pass per segment, once
      std::lock_guard<std::mutex> lk(g->layout_mu);
      if (!g->have_sync) {
        g->bv_sync.alloc((size_t)ng * sizeof(DecSync));
        bv_sync_index<<<(unsigned)((g->nseg + tpb - 1) / tpb), tpb, 0, st>>>(s, deg.as<uint32_t>(),
                                                                            g->bv_sync.as<DecSync>(), err.as<int>());
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (herr) throw AbiError(CMVG_ERR_CORRUPT, "BV stream corrupt (device index pass, code " + std::to_string(herr) + ")");
        g->have_sync = true;
      }
    }
    StreamScratch rbit(g->device, (size_t)g->n * 8, st), gcnt(g->device, (size_t)ng * 8, st),
        gbase(g->device, (size_t)ng * 8, st);
    bv_index_groups<<<(ng + 127) / 128, 128, 0, st>>>(s, g->bv_sync.as<DecSync>(), deg.as<uint32_t>(),
                                                      rbit.as<uint64_t>(), gcnt.as<uint64_t>(), err.as<int>());
    CUDA_TRY(cudaGetLastError());
    bv_scan_segments<<<1, 1024, 0, st>>>(gcnt.as<uint64_t>(), ng, kDecTileRows / kDecGroup, g->m,
                                         gbase.as<uint64_t>(), err.as<int>());
    CUDA_TRY(cudaGetLastError());
    // staging words (rows decoded into shared memory, references read from
    // there): off by default -- four CTAs per SM reading references through
    // L1/L2 beat two staged ones (C2 11.2 vs 15.8 ms)
    uint32_t cap = 0;
    if (const char* e = getenv("CMVG_DECODE_CAP")) cap = (uint32_t)strtoul(e, nullptr, 10);
    const uint32_t sm = dec_smem_bytes(cap);
    if (g->decode_attr < sm) {
      CUDA_TRY(cudaFuncSetAttribute(bv_decode_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      g->decode_attr = sm;
    }
    const uint32_t ntile = (uint32_t)(((uint64_t)g->n + kDecTileRows - 1) / kDecTileRows);
    bv_decode_tiles<<<ntile, kDecThreads, sm, st>>>(s, deg.as<uint32_t>(), rbit.as<uint64_t>(), gbase.as<uint64_t>(),
                                                    cap, ro, co, err.as<int>(), ref_out);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (herr) throw AbiError(CMVG_ERR_CORRUPT, "BV stream corrupt (device decode pass, code " + std::to_string(herr) + ")");
}
}  // namespace cmvg

extern "C" {

const char* cmvg_last_error(void) { return g_last_error.c_str(); }

// ---- host CSR --------------------------------------------------------------
int cmvg_csr_from_arrays(uint32_t n, const uint64_t* ro, const uint32_t* cols, cmvg_csr** out) {
  return guarded([&] {
    require(out && ro, "null argument");
    auto c = std::make_unique<cmvg_csr>();
    c->g.n = n;
    c->g.row_offsets.assign(ro, ro + (size_t)n + 1);
    require(c->g.row_offsets[0] == 0, "row_offsets[0] must be 0");
    uint64_t m = c->g.row_offsets[n];
    for (uint32_t u = 0; u < n; ++u) require(c->g.row_offsets[u] <= c->g.row_offsets[u + 1], "row_offsets must be nondecreasing");
    c->g.cols.assign(cols, cols + m);
    for (uint32_t u = 0; u < n; ++u)
      for (uint64_t e = c->g.row_offsets[u]; e < c->g.row_offsets[u + 1]; ++e) {
        if (c->g.cols[e] >= n) throw std::out_of_range("column " + std::to_string(c->g.cols[e]) + " >= n in row " + std::to_string(u));
        require(e == c->g.row_offsets[u] || c->g.cols[e] > c->g.cols[e - 1], "rows must be strictly increasing");
      }
    *out = c.release();
  });
}

int cmvg_gen_copy_model(uint32_t n, double mean_degree, double p_ref, double p_copy, uint64_t seed, cmvg_csr** out) {
  return guarded([&] {
    require(out, "null argument");
    CopyModelParams p;
    p.n = n;
    p.mean_degree = mean_degree;
    p.p_ref = p_ref;
    p.p_copy = p_copy;
    p.seed = seed;
    auto c = std::make_unique<cmvg_csr>();
    c->g = generate_copy_model(p);
    *out = c.release();
  });
}

int cmvg_gen_social(uint32_t n, uint64_t seed, cmvg_csr** out) {
  return guarded([&] {
    require(out, "null argument");
    SocialParams p;
    p.n = n;
    p.seed = seed;
    auto c = std::make_unique<cmvg_csr>();
    c->g = generate_social(p);
    *out = c.release();
  });
}

int cmvg_csr_transpose(const cmvg_csr* g, cmvg_csr** out) {
  return guarded([&] {
    require(g && out, "null argument");
    auto c = std::make_unique<cmvg_csr>();
    c->g = transpose_csr(g->g);
    *out = c.release();
  });
}

uint32_t cmvg_csr_n(const cmvg_csr* g) { return g ? g->g.n : 0; }
uint64_t cmvg_csr_m(const cmvg_csr* g) { return g ? g->g.m() : 0; }
const uint64_t* cmvg_csr_row_offsets(const cmvg_csr* g) { return g ? g->g.row_offsets.data() : nullptr; }
const uint32_t* cmvg_csr_cols(const cmvg_csr* g) { return g ? g->g.cols.data() : nullptr; }
void cmvg_csr_free(cmvg_csr* g) { delete g; }

// ---- BV stream -------------------------------------------------------------
static BvParams to_params(const cmvg_bv_params* p) {
  BvParams q;
  if (p) {
    q.window = p->window;
    q.max_ref = p->max_ref;
    q.min_interval = p->min_interval;
    q.zeta_k = p->zeta_k;
    q.segment_rows = p->segment_rows;
  }
  require(q.window <= 255, "window must be <= 255");
  require(q.min_interval >= 2, "min_interval must be >= 2");
  require(q.zeta_k >= 2 && q.zeta_k <= 8, "zeta_k must be in [2, 8]");
  require(q.segment_rows >= 1, "segment_rows must be >= 1");
  return q;
}

int cmvg_bv_encode(const cmvg_csr* g, const cmvg_bv_params* p, cmvg_bvstream** out) {
  return guarded([&] {
    require(g && out, "null argument");
    auto s = std::make_unique<cmvg_bvstream>();
    s->s = bv_encode(g->g, to_params(p));
    *out = s.release();
  });
}

int cmvg_bv_from_words(uint32_t n, uint64_t m, const cmvg_bv_params* p, const uint32_t* words, uint64_t nbits,
                       const uint64_t* seg, cmvg_bvstream** out) {
  return guarded([&] {
    require(out && (words || nbits == 0) && seg, "null argument");
    auto s = std::make_unique<cmvg_bvstream>();
    BvStream& b = s->s;
    b.n = n;
    b.m = m;
    b.params = to_params(p);
    b.nbits = nbits;
    b.words.assign(words, words + (nbits + 31) / 32);
    b.words.push_back(0);
    b.words.push_back(0);
    uint64_t nseg = ((uint64_t)n + b.params.segment_rows - 1) / b.params.segment_rows;
    b.segment_bit_offsets.assign(seg, seg + nseg + 1);
    if (b.segment_bit_offsets[nseg] != nbits) throw std::runtime_error("BV stream corrupt: segment table does not end at nbits");
    b.stats.stream_bits = nbits;
    *out = s.release();
  });
}

int cmvg_bv_save(const cmvg_bvstream* s, const char* path) {
  return guarded([&] {
    require(s && path, "null argument");
    save_bv_container(s->s, path);
  });
}

int cmvg_bv_load(const char* path, cmvg_bvstream** out) {
  return guarded([&] {
    require(path && out, "null argument");
    auto s = std::make_unique<cmvg_bvstream>();
    s->s = load_bv_container(path);
    *out = s.release();
  });
}

int cmvg_bv_describe(const cmvg_bvstream* s, uint32_t* n, uint64_t* m, cmvg_bv_params* p) {
  return guarded([&] {
    require(s && n && m && p, "null argument");
    *n = s->s.n;
    *m = s->s.m;
    p->window = s->s.params.window;
    p->max_ref = s->s.params.max_ref;
    p->min_interval = s->s.params.min_interval;
    p->zeta_k = s->s.params.zeta_k;
    p->segment_rows = s->s.params.segment_rows;
  });
}

int cmvg_bv_serialize(const cmvg_bvstream* s, uint8_t* buf, uint64_t cap, uint64_t* size) {
  return guarded([&] {
    require(s && size, "null argument");
    const std::vector<uint8_t> b = encode_bv_container(s->s);
    *size = b.size();
    if (buf && cap >= b.size()) std::memcpy(buf, b.data(), b.size());
  });
}

int cmvg_bv_deserialize(const uint8_t* buf, uint64_t size, cmvg_bvstream** out) {
  return guarded([&] {
    require((buf || size == 0) && out, "null argument");
    auto s = std::make_unique<cmvg_bvstream>();
    s->s = decode_bv_container(buf, (size_t)size);
    *out = s.release();
  });
}

int cmvg_bv_reconstruct_row(const cmvg_bvstream* s, uint32_t i, uint32_t* cols, uint64_t cap, uint64_t* deg) {
  return guarded([&] {
    require(s && deg, "null argument");
    const std::vector<uint32_t> row = bv_reconstruct_row(s->s, i);
    *deg = row.size();
    if (cols) {
      require(cap >= row.size(), "reconstruct_row: output too small");
      std::copy(row.begin(), row.end(), cols);
    }
  });
}

int cmvg_bv_decode_host(const cmvg_bvstream* s, cmvg_csr** out) {
  return guarded([&] {
    require(s && out, "null argument");
    auto c = std::make_unique<cmvg_csr>();
    BvDecoded d = bv_decode(s->s);
    if (d.csr.m() != s->s.m) throw std::runtime_error("BV stream corrupt: edge count mismatch");
    c->g = std::move(d.csr);
    *out = c.release();
  });
}

int cmvg_bv_get_stats(const cmvg_bvstream* s, cmvg_bv_stats* o) {
  return guarded([&] {
    require(s && o, "null argument");
    const BvStats& t = s->s.stats;
    o->stream_bits = s->s.nbits;
    o->rows_with_ref = t.rows_with_ref;
    o->copied_edges = t.copied_edges;
    o->interval_edges = t.interval_edges;
    o->intervals = t.intervals;
    o->residual_edges = t.residual_edges;
    o->minus_edges = t.minus_edges;
    o->max_depth = t.max_depth;
    o->nsegments = (uint32_t)(s->s.segment_bit_offsets.size() - 1);
  });
}

const uint32_t* cmvg_bv_words(const cmvg_bvstream* s, uint64_t* nwords) {
  if (!s) return nullptr;
  if (nwords) *nwords = (s->s.nbits + 31) / 32;
  return s->s.words.data();
}
const uint64_t* cmvg_bv_segment_offsets(const cmvg_bvstream* s, uint64_t* count) {
  if (!s) return nullptr;
  if (count) *count = s->s.segment_bit_offsets.size();
  return s->s.segment_bit_offsets.data();
}
void cmvg_bv_free(cmvg_bvstream* s) { delete s; }

// ---- device handle ----------------------------------------------------------
static void fill_bvt_info(cmvg_graph_info* o, const BvtStats& t) {
  o->bvt_stream_bytes = t.stream_bytes;
  o->bvt_entries = t.entries;
  o->bvt_far_slots = t.far_slots;
  o->bvt_heavy_targets = t.heavy_targets;
  o->bvt_slices = t.slices;
}
static void fill_bvf_info(cmvg_graph_info* o, const BvfStats& f) {
  o->bvf_stream_bytes = f.stream_bytes;
  o->bvf_terms = f.terms;
  o->bvf_pad_terms = f.pad_terms;
  o->bvf_slot_terms = f.slot_terms;
  o->bvf_esc_terms = f.esc_terms;
  o->bvf_esc_blocks = f.esc_blocks;
  o->bvf_max_K = f.max_K;
  o->bvf_min_cbits = f.min_cbits;
}
static void fill_bvs_info(cmvg_graph_info* o, const BvsStats& st, uint32_t cap) {
  o->bvs_stream_bytes = st.stream_bytes;
  o->bvs_max_block_words = st.max_block_words;
  o->bvs_stream_cap_words = cap;
  o->bvs_p995_block_words = st.p995_block_words;
  o->bvs_slices = st.slices;
  o->bvs_heavy_rows = st.heavy_rows;
  o->bvs_lane_words = st.lane_words;
  o->bvs_lane_words_used = st.lane_words_used;
  o->bvs_lane_iters = st.lane_iters;
  o->bvs_lane_iters_used = st.lane_iters_used;
}
void cmvg_default_opts(cmvg_create_opts* o) {
  if (!o) return;
  o->device = 0;
  o->block_rows = 1024;
  o->lanes = 256;
  o->window = 1536;
  o->stream_cap_words = 0;
  o->interval_mode = CMVG_INTERVALS_PREFIX;
  o->row_begin = 0;
  o->row_end = 0;
}

}  // extern "C"

// Copy this shard's slice of the host-built layouts to the device.
static void upload_layouts(cmvg_graph* g, BvdLayout& L, bool s, bool t, bool f) {
  const uint32_t bb = g->block_begin, be = g->block_begin + g->nblocks;
  if (s) {
    const uint64_t s0 = L.sblocks[bb].word_offset;
    const uint64_t s1 = L.sblocks[be - 1].word_offset + L.sblocks[be - 1].nwords;
    std::vector<BvdBlockInfo> sbl(L.sblocks.begin() + bb, L.sblocks.begin() + be);
    for (auto& b : sbl) b.word_offset -= s0;
    std::vector<uint32_t> sw(L.swords.begin() + s0, L.swords.begin() + s1);
    sw.resize(sw.size() + 2 * kBvsGuardWords, 0);
    g->swords.upload(sw.data(), sw.size());
    g->sblocks.upload(sbl.data(), sbl.size());
    g->heavy_items = L.sstats.heavy_chunks;
    g->s_stream_bytes = (s1 - s0) * 4;
    g->sstats = L.sstats;
    g->have_bvs = true;
  }
  if (t) {
    const uint64_t t0 = L.tblocks[bb].word_offset;
    const uint64_t t1 = L.tblocks[be - 1].word_offset + L.tblocks[be - 1].nwords;
    std::vector<BvdBlockInfo> tbl(L.tblocks.begin() + bb, L.tblocks.begin() + be);
    for (auto& b : tbl) b.word_offset -= t0;
    std::vector<uint32_t> tw(L.twords.begin() + t0, L.twords.begin() + t1);
    tw.resize(tw.size() + 64, 0);
    g->twords.upload(tw.data(), tw.size());
    g->tblocks.upload(tbl.data(), tbl.size());
    g->t_stream_bytes = (t1 - t0) * 4;
    g->tstats = L.tstats;
    g->tfar_begin = L.tblocks[bb].pad[0];
    g->tfar_end = be < L.tblocks.size() ? L.tblocks[be].pad[0] : (uint32_t)L.tstats.far_slots;
    g->tile_ptr.upload(L.tile_ptr.data(), L.tile_ptr.size());
    g->tile_blk.upload(L.tile_blk.data(), std::max<size_t>(1, L.tile_blk.size()));
    g->farp_ptr.upload(L.farp_ptr.data(), L.farp_ptr.size());
    if (L.farp.empty()) L.farp.assign(2, 0u);
    g->farp.upload(L.farp.data(), L.farp.size());
    g->have_bvt = true;
  }
  if (f) {
    const uint64_t f0 = L.fblocks[bb].word_offset;
    const uint64_t f1 = L.fblocks[be - 1].word_offset + L.fblocks[be - 1].nwords;
    std::vector<BvfBlockInfo> fbl(L.fblocks.begin() + bb, L.fblocks.begin() + be);
    for (auto& b : fbl) b.word_offset -= f0;
    std::vector<uint32_t> fw(L.fwords.begin() + f0, L.fwords.begin() + f1);
    fw.resize(fw.size() + 64, 0);
    g->fwords.upload(fw.data(), fw.size());
    g->fblocks.upload(fbl.data(), fbl.size());
    {  // flat escape columns (the pre-gather's index list)
      std::vector<uint32_t> ec, eb(fbl.size() + 1, 0);
      g->fesc_base_h.assign(fbl.size() + 1, 0);
      for (size_t q = 0; q < fbl.size(); ++q) {
        const BvfBlockInfo& b = fbl[q];
        if (b.flags & kBvfFlagEsc) {
          const uint32_t* es = fw.data() + b.word_offset + b.esc_off;
          const uint32_t ne = es[b.nact];
          const uint32_t* cols = es + bvf_align4(b.nact + 1u);
          ec.insert(ec.end(), cols, cols + ne);
        }
        if (ec.size() > 0xffffffffull) throw std::runtime_error("BV-F: more than 2^32 escape terms in one shard");
        eb[q + 1] = (uint32_t)ec.size();
        g->fesc_base_h[q + 1] = ec.size();
      }
      ec.resize(ec.size() + 4, 0u);
      g->fesc.upload(ec.data(), ec.size());
      g->fesc_base.upload(eb.data(), eb.size());
    }
    g->f_stream_bytes = (f1 - f0) * 4;
    g->fstats = L.fstats;
  }
}

namespace cmvg {
// The sliced (matmat) and target-sorted (scatter) layouts are built on their
// first use: a handle that only gathers (A x, PageRank) never pays for them.
void ensure_layouts(cmvg_graph* g, bool s, bool t) {
  if ((!s || g->have_bvs) && (!t || g->have_bvt)) return;
  std::lock_guard<std::mutex> lk(g->layout_mu);
  s = s && !g->have_bvs;
  t = t && !g->have_bvt;
  if (!s && !t) return;
  BvDecoded dec = bv_decode(*g->host_stream);
  BvdOptions bo = g->build_opts;
  bo.bvs = s;
  bo.bvt = t;
  bo.bvf = false;
  BvdLayout L = build_bvd(dec, g->host_stream->params, bo);
  DeviceGuard dg(g->device);
  upload_layouts(g, L, s, t, false);
}
}  // namespace cmvg

extern "C" {

int cmvg_create(const cmvg_bvstream* s, const cmvg_create_opts* opts_in, cmvg_graph** out) {
  return guarded([&] {
    require(s && out, "null argument");
    cmvg_create_opts o;
    cmvg_default_opts(&o);
    if (opts_in) o = *opts_in;
    const BvStream& bs = s->s;
    require(bs.params.window <= 7, "the device layout supports BV windows w <= 7");
    require(bs.params.zeta_k == 3, "device kernels support zeta_3 residuals");
    require(bs.n > 0, "empty graph");
    require(o.lanes >= 32 && o.lanes <= 256 && (o.lanes & (o.lanes - 1)) == 0,
            "lanes (threads per block) must be a power of two in [32, 256]");
    require(o.block_rows <= 4 * o.lanes, "block_rows must be <= 4 x threads per block");
    require(o.window <= 3968, "window must be <= 3968 entries (the 13-bit BV-F term index)");
    require(o.interval_mode <= CMVG_INTERVALS_DIRECT, "bad interval_mode");
    uint32_t row_end = o.row_end ? o.row_end : bs.n;
    require(o.row_begin < row_end && row_end <= bs.n, "bad shard row range");
    require(o.row_begin % o.block_rows == 0, "shard row_begin must be a multiple of block_rows");
    require(row_end == bs.n || row_end % o.block_rows == 0, "shard row_end must be a multiple of block_rows or n");

    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    require(o.device >= 0 && o.device < ndev, "no such CUDA device");

    BvdOptions bo;
    bo.block_rows = o.block_rows;
    bo.window = o.window;
    bo.bvs = false;  // the sliced (matmat) and target-sorted (scatter) layouts are built on first use
    bo.bvt = false;
    const uint32_t B = o.block_rows;
    require(B && !(B & (B - 1)) && B % bs.params.segment_rows == 0 && B <= 1024,
            "block_rows must be a power of two <= 1024 and a multiple of the BV segment");
    require(o.window % 16 == 0 && o.window > 0, "window must be a positive multiple of 16");

    auto g = std::make_unique<cmvg_graph>();
    g->device = o.device;
    g->n = bs.n;
    g->m = bs.m;
    g->params = bs.params;
    g->row_begin = o.row_begin;
    g->row_end = row_end;
    g->block_begin = o.row_begin / o.block_rows;
    const uint32_t block_end = (uint32_t)(((uint64_t)row_end + o.block_rows - 1) / o.block_rows);
    g->nblocks = block_end - g->block_begin;
    g->interval_mode = o.interval_mode;
    g->threads = o.lanes;
    g->bv_bits = bs.nbits;
    g->nseg = bs.segment_bit_offsets.size() - 1;
    static const bool timing = getenv("CMVG_BUILD_TIMING") != nullptr;
    auto tc0 = std::chrono::steady_clock::now();
    g->host_stream = s->sp;
    g->build_opts = bo;
    DeviceGuard dg(o.device);
    g->bv_words.upload(bs.words.data(), bs.words.size());
    g->bv_seg.upload(bs.segment_bit_offsets.data(), bs.segment_bit_offsets.size());
    if (timing)
      fprintf(stderr, "[create] stream copy + upload %.2f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc0).count());

    // the BV-F layout: built on the GPU from the BV stream (bvf_build.cu), or
    // on the host (CMVG_HOST_BUILD=1, and streams the tile decoder cannot serve)
    bool built = false;
    if (!getenv("CMVG_HOST_BUILD")) {
      g->dims = BvdDims{bs.n, o.block_rows, o.window, bs.params.min_interval,
                        (uint32_t)(((uint64_t)bs.n + o.block_rows - 1) / o.block_rows), 0, 0, 0};
      DeviceBuildStats ds;
      bool ok = false;
      try {
        ok = device_build_bvf(g.get(), 0, ds);
      } catch (const AbiError& e) {
        if (e.code != CMVG_ERR_NOMEM) throw;  // a corrupt stream stays an error
        (void)cudaGetLastError();
        g->fwords.free_now();
        g->fesc.free_now();
        ok = false;  // not enough device memory for the build's arenas: the host build below
      }
      if (ok) {
        built = true;
        g->device_built = true;
        g->adds = ds.adds;
        g->stats.window_coverage = ds.window_coverage;
        g->stream_cap_words = o.stream_cap_words ? o.stream_cap_words : 1024u;
      }
    }
    if (!built) {
      BvDecoded dec = bv_decode(bs);
      if (dec.csr.m() != bs.m) throw std::runtime_error("BV stream corrupt: edge count mismatch");
      BvdLayout L = build_bvd(dec, bs.params, bo);
      g->dims = L.dims;
      g->stream_cap_words = o.stream_cap_words ? o.stream_cap_words
                                               : std::min<uint32_t>(12288, std::max<uint32_t>(1024, (L.stats.p995_block_words + 255) & ~255u));
      g->stats.codes = L.stats.codes;
      g->stats.window_coverage = L.stats.window_coverage;
      g->stats.p995_block_words = L.stats.p995_block_words;
      {  // read set: the blocks' x-windows and their out-of-window columns (bitmap, O(n))
        std::vector<uint64_t> bm(((uint64_t)bs.n + 63) / 64, 0);
        auto mark = [&](uint64_t c) { bm[c >> 6] |= 1ull << (c & 63); };
        for (uint32_t b = g->block_begin; b < block_end; ++b) {
          const uint64_t w0 = L.blocks[b].wlo, w1 = std::min<uint64_t>(bs.n, w0 + L.dims.window);
          for (uint64_t c = w0; c < w1; ++c) mark(c);
          for (uint64_t q = L.rfar_ptr[b]; q < L.rfar_ptr[b + 1]; ++q) mark(L.rfar[q]);
        }
        std::vector<uint32_t>& rs = g->read_set;
        rs.clear();
        for (uint64_t wi = 0; wi < bm.size(); ++wi)
          for (uint64_t v = bm[wi]; v; v &= v - 1) rs.push_back((uint32_t)(wi * 64 + __builtin_ctzll(v)));
        g->have_read_set = true;
      }
      g->win_need.resize(g->nblocks);
      g->far_need.resize(g->nblocks);
      {
        uint64_t pm = 0, fm = 0;
        for (uint32_t q = 0; q < g->nblocks; ++q) {
          const uint32_t b = g->block_begin + q;
          pm = std::max<uint64_t>(pm, (uint64_t)L.blocks[b].wlo + L.dims.window);
          g->win_need[q] = (uint32_t)std::min<uint64_t>(pm, bs.n);
          for (uint64_t r = L.rfar_ptr[b]; r < L.rfar_ptr[b + 1]; ++r) fm = std::max<uint64_t>(fm, (uint64_t)L.rfar[r] + 1);
          g->far_need[q] = (uint32_t)std::min<uint64_t>(fm, bs.n);
        }
      }
      upload_layouts(g.get(), L, false, false, true);
      // stats of the shard
      const uint64_t w0 = L.blocks[g->block_begin].word_offset;
      const uint64_t w1 = L.blocks[block_end - 1].word_offset + L.blocks[block_end - 1].nwords;
      g->stats.stream_bytes = (w1 - w0) * 4;
      g->stats.block_table_bytes = (uint64_t)g->nblocks * sizeof(BvdBlockInfo);
      g->stats.row_bits = L.stats.row_bits;  // whole graph
      g->adds = L.adds_per_product;
    }
    *out = g.release();
  });
}

int cmvg_layout_info(const cmvg_bvstream* s, const cmvg_create_opts* opts_in, cmvg_graph_info* o) {
  return guarded([&] {
    require(s && o, "null argument");
    cmvg_create_opts opt;
    cmvg_default_opts(&opt);
    if (opts_in) opt = *opts_in;
    const BvStream& bs = s->s;
    BvDecoded dec = bv_decode(bs);
    BvdOptions bo;
    bo.block_rows = opt.block_rows;
    bo.window = opt.window;
    BvdLayout L = build_bvd(dec, bs.params, bo);
    std::memset(o, 0, sizeof(*o));
    o->n = bs.n;
    o->m = bs.m;
    o->row_begin = 0;
    o->row_end = bs.n;
    o->bv_stream_bits = bs.nbits;
    o->bvd_row_bits = L.stats.row_bits;
    o->bvd_stream_bytes = L.stats.stream_bytes;
    o->bvd_lane_table_bytes = 0;
    o->bvd_block_table_bytes = L.stats.block_table_bytes;
    o->block_rows = L.dims.block_rows;
    o->lanes = opt.lanes;
    o->window = L.dims.window;
    o->nblocks = L.dims.nblocks;
    o->max_depth = L.dims.max_depth;
    o->interval_mode = opt.interval_mode;
    o->adds_per_product = L.adds_per_product;
    o->device_bytes = 0;
    o->bvd_codes = L.stats.codes;
    o->max_block_words = L.dims.max_block_words;
    o->stream_cap_words = opt.stream_cap_words
                              ? opt.stream_cap_words
                              : std::min<uint32_t>(12288, std::max<uint32_t>(1024, (L.stats.p995_block_words + 255) & ~255u));
    o->window_coverage = L.stats.window_coverage;
    fill_bvs_info(o, L.sstats, 0);
    fill_bvt_info(o, L.tstats);
    fill_bvf_info(o, L.fstats);
  });
}

int cmvg_layout_export(const cmvg_bvstream* s, const cmvg_create_opts* opts_in, cmvg_layout** out) {
  return guarded([&] {
    require(s && out, "null argument");
    cmvg_create_opts opt;
    cmvg_default_opts(&opt);
    if (opts_in) opt = *opts_in;
    BvDecoded dec = bv_decode(s->s);
    BvdOptions bo;
    bo.block_rows = opt.block_rows;
    bo.window = opt.window;
    auto l = std::make_unique<cmvg_layout>();
    l->L = build_bvd(dec, s->s.params, bo);
    *out = l.release();
  });
}
const uint32_t* cmvg_layout_words(const cmvg_layout* l, uint64_t* nwords) {
  if (!l) return nullptr;
  if (nwords) *nwords = l->L.words.size();
  return l->L.words.data();
}
const uint32_t* cmvg_layout_blocks(const cmvg_layout* l, uint32_t* nblocks) {
  static_assert(sizeof(BvdBlockInfo) == 32, "block info is 8 u32");
  if (!l) return nullptr;
  if (nblocks) *nblocks = (uint32_t)l->L.blocks.size();
  return reinterpret_cast<const uint32_t*>(l->L.blocks.data());
}
const uint32_t* cmvg_layout_swords(const cmvg_layout* l, uint64_t* nwords) {
  if (!l) return nullptr;
  if (nwords) *nwords = l->L.swords.size();
  return l->L.swords.data();
}
const uint32_t* cmvg_layout_sblocks(const cmvg_layout* l, uint32_t* nblocks) {
  if (!l) return nullptr;
  if (nblocks) *nblocks = (uint32_t)l->L.sblocks.size();
  return reinterpret_cast<const uint32_t*>(l->L.sblocks.data());
}
const uint32_t* cmvg_layout_twords(const cmvg_layout* l, uint64_t* nwords) {
  if (!l) return nullptr;
  if (nwords) *nwords = l->L.twords.size();
  return l->L.twords.data();
}
const uint32_t* cmvg_layout_tblocks(const cmvg_layout* l, uint32_t* nblocks) {
  if (!l) return nullptr;
  if (nblocks) *nblocks = (uint32_t)l->L.tblocks.size();
  return reinterpret_cast<const uint32_t*>(l->L.tblocks.data());
}
const uint32_t* cmvg_layout_fwords(const cmvg_layout* l, uint64_t* nwords) {
  if (!l) return nullptr;
  if (nwords) *nwords = l->L.fwords.size();
  return l->L.fwords.data();
}
const uint32_t* cmvg_layout_fblocks(const cmvg_layout* l, uint32_t* nblocks) {
  if (!l) return nullptr;
  if (nblocks) *nblocks = (uint32_t)l->L.fblocks.size();
  return reinterpret_cast<const uint32_t*>(l->L.fblocks.data());
}
void cmvg_layout_free(cmvg_layout* l) { delete l; }

int cmvg_destroy(cmvg_graph* g) {
  if (!g) return CMVG_OK;
  {
    DeviceGuard dg(g->device);
    delete g;
  }
  return CMVG_OK;
}

int cmvg_graph_info_get(const cmvg_graph* g, cmvg_graph_info* o) {
  return guarded([&] {
    require(g && o, "null argument");
    std::memset(o, 0, sizeof(*o));
    o->n = g->n;
    o->m = g->m;
    o->row_begin = g->row_begin;
    o->row_end = g->row_end;
    o->bv_stream_bits = g->bv_bits;
    o->bvd_row_bits = g->stats.row_bits;
    o->bvd_stream_bytes = g->stats.stream_bytes;
    o->bvd_lane_table_bytes = 0;
    o->bvd_block_table_bytes = g->stats.block_table_bytes;
    o->block_rows = g->dims.block_rows;
    o->lanes = g->threads;
    o->window = g->dims.window;
    o->nblocks = g->nblocks;
    o->max_depth = g->dims.max_depth;
    o->interval_mode = g->interval_mode;
    o->adds_per_product = g->adds;
    o->device_bytes = g->device_bytes();
    o->bvd_codes = g->stats.codes;
    o->max_block_words = g->dims.max_block_words;
    o->stream_cap_words = g->stream_cap_words;
    o->window_coverage = g->stats.window_coverage;
    fill_bvs_info(o, g->sstats, 0);
    o->bvs_stream_bytes = g->s_stream_bytes;
    fill_bvt_info(o, g->tstats);
    o->bvt_stream_bytes = g->t_stream_bytes;
    fill_bvf_info(o, g->fstats);
    o->bvf_stream_bytes = g->f_stream_bytes;
  });
}

int cmvg_bvf_export(const cmvg_graph* g, uint32_t* words, uint64_t words_cap, uint32_t* blocks, uint64_t blocks_cap,
                    uint64_t* nwords, uint32_t* nblocks, int* device_built) {
  return guarded([&] {
    require(g && nwords && nblocks, "null argument");
    *nwords = g->f_stream_bytes / 4;
    *nblocks = g->nblocks;
    if (device_built) *device_built = g->device_built ? 1 : 0;
    DeviceGuard dg(g->device);
    if (words && words_cap >= *nwords && *nwords)
      CUDA_TRY(cudaMemcpy(words, g->fwords.p, *nwords * 4, cudaMemcpyDeviceToHost));
    if (blocks && blocks_cap >= (uint64_t)*nblocks * 8)
      CUDA_TRY(cudaMemcpy(blocks, g->fblocks.p, (size_t)*nblocks * sizeof(BvfBlockInfo), cudaMemcpyDeviceToHost));
  });
}

int cmvg_read_set(const cmvg_graph* g, uint32_t* cols, uint64_t cap, uint64_t* count) {
  return guarded([&] {
    require(g && count, "null argument");
    ensure_read_set(g);
    *count = g->read_set.size();
    if (cols && cap >= g->read_set.size()) std::memcpy(cols, g->read_set.data(), g->read_set.size() * 4);
  });
}

uint32_t cmvg_dimension(const cmvg_graph* g) { return g ? g->n : 0; }
uint64_t cmvg_adds_per_product(const cmvg_graph* g) { return g ? g->adds : 0; }

}  // extern "C"

// ---------------------------------------------------------------------------
// kernel launches
namespace {

template <typename XT, typename YT>
void launch_gather(cmvg_graph* g, const XT* x, YT* y, cudaStream_t st, const XT* xfar = nullptr, uint32_t b0 = 0,
                   uint32_t b1 = 0xffffffffu) {
  launch_bvf<XT, YT, false>(g, x, xfar, y, PrArgs{}, st, b0, b1);
}

// Mapped device address of a pinned host buffer, or nullptr (pageable memory).
const void* mapped_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Pipelined host-pointer gather (pinned x and y): x is uploaded in chunks in
// row order; blocks run as soon as their x-window has arrived, reading the
// rare columns outside the window (`far`) straight from the mapped host x;
// each chunk's y rows go back while later chunks upload -- H2D, compute and
// D2H overlap across chunks (PCIe is full duplex).
// Host memcpy over `threads` threads (pageable <-> pinned staging).
void par_copy(void* dst, const void* src, size_t bytes, unsigned threads) {
  if (bytes < (size_t(1) << 20) || threads <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t part = ((bytes + threads - 1) / threads + 63) & ~size_t(63);
  std::vector<std::thread> th;
  for (unsigned t = 1; t < threads && (size_t)t * part < bytes; ++t) {
    const size_t a = (size_t)t * part, b = std::min(bytes, a + part);
    th.emplace_back([=] { std::memcpy((char*)dst + a, (const char*)src + a, b - a); });
  }
  std::memcpy(dst, src, std::min(bytes, part));
  for (auto& t : th) t.join();
}

// ux / uy (pageable x and y): x and y are then the handle's pinned staging
// buffers; each chunk's x range is copied ux -> x just before its upload, and
// a second host thread copies each chunk's y rows y -> uy as soon as their
// download completes, so the host copies overlap the transfers and kernels.
template <typename T>
void gather_host_pipelined(cmvg_graph* g, const T* x, T* y, const T* xmapped, const T* ux = nullptr, T* uy = nullptr) {
  const uint32_t nb = g->nblocks, B = g->dims.block_rows;
  // chunk boundaries (in blocks): a ramp up (1/4, 1/2, 3/4 of a chunk: the
  // first D2H starts early), equal chunks, then 1/2, 1/4, 1/8, 1/8 (a short
  // last chunk keeps the tail -- last kernel + last D2H -- small)
  const uint32_t C = std::min<uint32_t>(16, nb);  // 2 events per chunk: g->ev has 32
  std::vector<uint32_t> cut(C + 1, 0);
  {
    static const double w[16] = {0.25, 0.5, 0.75, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0.5, 0.25, 0.125, 0.125};
    double tot = 0.0, acc = 0.0;
    for (uint32_t c = 0; c < C; ++c) tot += C == 16 ? w[c] : 1.0;
    for (uint32_t c = 0; c < C; ++c) {
      acc += C == 16 ? w[c] : 1.0;
      cut[c + 1] = std::min<uint32_t>(nb, (uint32_t)((double)nb * acc / tot + 0.5));
    }
    cut[C] = nb;
    for (uint32_t c = 1; c <= C; ++c) cut[c] = std::max(cut[c], cut[c - 1]);
  }
  if (!g->s_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&g->s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&g->s_comp, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&g->s_out, cudaStreamNonBlocking));
    for (int i = 0; i < 32; ++i) CUDA_TRY(cudaEventCreateWithFlags(&g->ev[i], cudaEventDisableTiming));
  }
  const size_t nrows = (size_t)g->row_end - g->row_begin;
  T* hx = g->hx.as<T>();
  T* hy = g->hy.as<T>();
  size_t xdone = 0;
  // CMVG_PIPE_TRACE=1 (dev): timing events per chunk, the timeline on stderr
  static const bool trace = std::getenv("CMVG_PIPE_TRACE") != nullptr;
  cudaEvent_t tev[3 * 16 + 1];
  if (trace) {
    for (auto& e : tev) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventRecord(tev[3 * 16], g->s_in));
  }
  // the last non-empty chunk uploads the rest of x
  uint32_t last = C - 1;
  while (last > 0 && cut[last] == cut[last + 1]) --last;
  const unsigned cth = std::max(1u, std::min(8u, host_threads() / 2));
  // pageable y: the chunks' download events, consumed by the y-copier thread
  std::vector<std::pair<size_t, size_t>> yrange(C, {0, 0});
  std::vector<cudaEvent_t> yev(C, nullptr);
  std::mutex ymu;
  std::condition_variable ycv;
  uint32_t yposted = 0;
  bool yabort = false;
  std::atomic<bool> yfail{false};
  std::thread ycopier;
  if (uy) {
    for (uint32_t c = 0; c < C; ++c) CUDA_TRY(cudaEventCreateWithFlags(&yev[c], cudaEventDisableTiming));
    ycopier = std::thread([&] {
      for (uint32_t c = 0; c < C; ++c) {
        {
          std::unique_lock<std::mutex> lk(ymu);
          ycv.wait(lk, [&] { return yabort || yposted > c; });
          if (yabort) return;
        }
        if (yrange[c].second > yrange[c].first) {
          if (cudaEventSynchronize(yev[c]) != cudaSuccess) {
            yfail = true;
            return;
          }
          par_copy(uy + yrange[c].first, y + yrange[c].first, (yrange[c].second - yrange[c].first) * sizeof(T), cth);
        }
      }
    });
  }
  auto post_y = [&](uint32_t c) {  // chunks < c may be copied out
    std::lock_guard<std::mutex> lk(ymu);
    yposted = c;
    ycv.notify_one();
  };
  try {
  for (uint32_t c = 0; c <= last; ++c) {
    const uint32_t b0 = cut[c], b1 = cut[c + 1];
    if (b0 == b1) continue;  // empty chunk (rounding of the chunk weights)
    // x needed by blocks < b1: their windows (prefix max) plus a lookahead
    // that covers most out-of-window columns (512 KB of fp64: ~10 us of
    // PCIe), everything for the last chunk
    constexpr size_t kLookahead = size_t(1) << 16;
    size_t need = c == last ? g->n : std::min<size_t>(g->n, g->win_need[b1 - 1] + kLookahead);
    if (need > xdone) {
      if (ux) par_copy(const_cast<T*>(x) + xdone, ux + xdone, (need - xdone) * sizeof(T), cth);
      CUDA_TRY(cudaMemcpyAsync(hx + xdone, x + xdone, (need - xdone) * sizeof(T), cudaMemcpyHostToDevice, g->s_in));
      xdone = need;
    }
    CUDA_TRY(cudaEventRecord(g->ev[2 * c], g->s_in));
    if (trace) CUDA_TRY(cudaEventRecord(tev[3 * c], g->s_in));
    CUDA_TRY(cudaStreamWaitEvent(g->s_comp, g->ev[2 * c], 0));
    // columns outside the blocks' windows: from the device copy when all of
    // them are already uploaded (the lookahead makes that the common case),
    // else from the mapped host x -- PCIe round trips that queue behind the
    // H2D stream
    const bool far_on_device = g->far_need.empty() || g->far_need[b1 - 1] <= xdone;
    if (trace && !far_on_device) std::fprintf(stderr, "chunk %2u: far columns from mapped host x\n", c);
    launch_gather<T, T>(g, hx, hy, g->s_comp, far_on_device ? hx : xmapped, b0, b1);
    CUDA_TRY(cudaEventRecord(g->ev[2 * c + 1], g->s_comp));
    if (trace) CUDA_TRY(cudaEventRecord(tev[3 * c + 1], g->s_comp));
    CUDA_TRY(cudaStreamWaitEvent(g->s_out, g->ev[2 * c + 1], 0));
    const size_t r0 = std::min(nrows, (size_t)b0 * B), r1 = std::min(nrows, (size_t)b1 * B);
    if (r1 > r0) CUDA_TRY(cudaMemcpyAsync(y + r0, hy + r0, (r1 - r0) * sizeof(T), cudaMemcpyDeviceToHost, g->s_out));
    if (trace) CUDA_TRY(cudaEventRecord(tev[3 * c + 2], g->s_out));
    if (uy) {
      yrange[c] = {r0, r1};
      CUDA_TRY(cudaEventRecord(yev[c], g->s_out));
      post_y(c + 1);
    }
  }
  if (uy) post_y(C);
  } catch (...) {
    // copies already queued must not outlive the call (they read the caller's buffers)
    (void)cudaStreamSynchronize(g->s_in);
    (void)cudaStreamSynchronize(g->s_comp);
    (void)cudaStreamSynchronize(g->s_out);
    if (uy) {
      {
        std::lock_guard<std::mutex> lk(ymu);
        yabort = true;
      }
      ycv.notify_one();
      ycopier.join();
      for (auto& e : yev) cudaEventDestroy(e);
    }
    throw;
  }
  CUDA_TRY(cudaStreamSynchronize(g->s_out));
  if (uy) {
    ycopier.join();
    for (auto& e : yev) cudaEventDestroy(e);
    if (yfail) throw AbiError(CMVG_ERR_CUDA, "pipelined host gather: a download failed");
  }
  if (trace) {
    for (uint32_t c = 0; c < C; ++c) {
      float a = 0, b = 0, d = 0;
      if (cudaEventElapsedTime(&a, tev[3 * 16], tev[3 * c]) != cudaSuccess ||
          cudaEventElapsedTime(&b, tev[3 * 16], tev[3 * c + 1]) != cudaSuccess ||
          cudaEventElapsedTime(&d, tev[3 * 16], tev[3 * c + 2]) != cudaSuccess) {
        (void)cudaGetLastError();  // a skipped (empty) chunk
        continue;
      }
      std::fprintf(stderr, "chunk %2u blocks [%u,%u) h2d_end %.3f kern_end %.3f d2h_end %.3f ms\n", c, cut[c],
                   cut[c + 1], a, b, d);
    }
    for (auto& e : tev) cudaEventDestroy(e);
  }
}

// the A^T handle of g (CMVG_LEFT), built on first use
cmvg_graph* ensure_left(cmvg_graph* g) {
  std::lock_guard<std::mutex> lk(g->left_mu);
  if (!g->left) g->left = build_left_handle(g, 0);
  return g->left.get();
}

template <typename T>
int matvec_impl(cmvg_graph* g, const T* x, T* y, int form, int ptr_kind, void* stream) {
  return guarded([&] {
    require(g && x && y, "null argument");
    require(form == CMVG_GATHER || form == CMVG_SCATTER || form == CMVG_LEFT, "bad form");
    require(ptr_kind == CMVG_HOST || ptr_kind == CMVG_DEVICE, "bad ptr_kind");
    if (form == CMVG_LEFT) {  // x A = (A^T) x: the gather on the transpose's layout
      require(g->row_begin == 0 && g->row_end == g->n, "x A (CMVG_LEFT) needs a whole-graph handle");
      DeviceGuard dg0(g->device);
      g = ensure_left(g);
      form = CMVG_GATHER;
    }
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t nin = g->n;
    const size_t nout = form == CMVG_GATHER ? (size_t)(g->row_end - g->row_begin) : (size_t)g->n;
    auto run = [&](const T* dx, T* dy) {
      if (form == CMVG_GATHER) launch_gather<T, T>(g, dx, dy, st);
      else launch_scatter<T>(g, dx, dy, st);
    };
    if (ptr_kind == CMVG_DEVICE) {
      require(aligned16(x) && aligned16(y), "device buffers must be 16-byte aligned");
      run(x, y);
      return;
    }
    std::lock_guard<std::mutex> lk(g->host_mu);
    g->hx.alloc(nin * sizeof(T) + 64);
    g->hy.alloc(nout * sizeof(T) + 64);
    if (form == CMVG_GATHER) {
      const T* xm = static_cast<const T*>(mapped_host(x));
      if (st) CUDA_TRY(cudaStreamSynchronize(st));  // the caller's prior work on x / y
      if (xm && mapped_host(y)) {
        gather_host_pipelined<T>(g, x, y, xm);
        return;
      }
      // pageable (std::vector spans, numpy arrays): the same pipeline through
      // the handle's pinned staging buffers, host copies overlapped
      g->px.alloc(nin * sizeof(T) + 64);
      g->py.alloc(nout * sizeof(T) + 64);
      const T* pxm = static_cast<const T*>(mapped_host(g->px.p));
      gather_host_pipelined<T>(g, g->px.as<T>(), g->py.as<T>(), pxm, x, y);
      return;
    }
    CUDA_TRY(cudaMemcpyAsync(g->hx.p, x, nin * sizeof(T), cudaMemcpyHostToDevice, st));
    run(g->hx.as<T>(), g->hy.as<T>());
    CUDA_TRY(cudaMemcpyAsync(y, g->hy.p, nout * sizeof(T), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  });
}

}  // namespace

extern "C" {

int cmvg_matvec_f64(cmvg_graph* g, const double* x, double* y, int form, int ptr_kind, void* stream) {
  return matvec_impl<double>(g, x, y, form, ptr_kind, stream);
}
int cmvg_matvec_f32(cmvg_graph* g, const float* x, float* y, int form, int ptr_kind, void* stream) {
  return matvec_impl<float>(g, x, y, form, ptr_kind, stream);
}

int cmvg_matmat_f32(cmvg_graph* g, const float* X, float* Y, uint32_t k, int ptr_kind, void* stream) {
  return guarded([&] {
    require(g && X && Y, "null argument");
    require(k >= 1, "k must be >= 1");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t nin = (size_t)g->n * k, nout = (size_t)(g->row_end - g->row_begin) * k;
    if (ptr_kind == CMVG_DEVICE) {
      launch_matmat(g, X, Y, k, st);
      return;
    }
    std::lock_guard<std::mutex> lk(g->host_mu);
    g->hx.alloc(nin * 4 + 64);
    g->hy.alloc(nout * 4 + 64);
    CUDA_TRY(cudaMemcpyAsync(g->hx.p, X, nin * 4, cudaMemcpyHostToDevice, st));
    launch_matmat(g, g->hx.as<float>(), g->hy.as<float>(), k, st);
    CUDA_TRY(cudaMemcpyAsync(Y, g->hy.p, nout * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  });
}


int cmvg_decode_csr(cmvg_graph* g, uint64_t* row_offsets, uint32_t* cols, int ptr_kind, void* stream) {
  return guarded([&] {
    require(g && row_offsets && (cols || g->m == 0), "null argument");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf dro, dcols;
    uint64_t* ro = row_offsets;
    uint32_t* co = cols;
    if (ptr_kind == CMVG_HOST) {
      dro.alloc(((size_t)g->n + 1) * 8);
      dcols.alloc(g->m * 4 + 16);
      ro = dro.as<uint64_t>();
      co = dcols.as<uint32_t>();
    }
    decode_device(g, ro, co, nullptr, st);
    if (ptr_kind == CMVG_HOST) {
      CUDA_TRY(cudaMemcpyAsync(row_offsets, ro, ((size_t)g->n + 1) * 8, cudaMemcpyDeviceToHost, st));
      if (g->m) CUDA_TRY(cudaMemcpyAsync(cols, co, g->m * 4, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
    }
  });
}

int cmvg_pagerank_ex(cmvg_graph* g, const uint32_t* degrees, double alpha, uint32_t iterations, double l1_tolerance,
                     int dangling, const double* start, double* ranks, uint32_t* iterations_run, int ptr_kind,
                     void* stream) {
  return guarded([&] {
    require(g && degrees && ranks, "null argument");
    require(alpha > 0.0 && alpha < 1.0, "alpha must be in (0,1)");
    require(iterations > 0, "iterations must be > 0");
    require(dangling == CMVG_DANGLING_UNIFORM || dangling == CMVG_DANGLING_DROP, "bad dangling policy");
    require(g->row_begin == 0 && g->row_end == g->n, "cmvg_pagerank needs a whole-graph handle");
    DeviceGuard dg(g->device);
    if (start) {  // a probability vector (pagerank.hpp:97; the same check as the reference)
      std::vector<double> hs;
      const double* sp = start;
      if (ptr_kind == CMVG_DEVICE) {
        hs.resize(g->n);
        CUDA_TRY(cudaMemcpy(hs.data(), start, (size_t)g->n * 8, cudaMemcpyDeviceToHost));
        sp = hs.data();
      }
      double sum = 0.0;
      for (uint32_t i = 0; i < g->n; ++i) {
        require(sp[i] >= 0.0, "pagerank: start has a negative entry");
        sum += sp[i];
      }
      require(std::fabs(sum - 1.0) <= 1e-9, "pagerank: start is not a probability vector");
    }
    run_pagerank(g, degrees, alpha, iterations, l1_tolerance, dangling, start, ranks, iterations_run, ptr_kind,
                 (cudaStream_t)stream);
  });
}

int cmvg_pagerank(cmvg_graph* g, const uint32_t* degrees, double alpha, uint32_t iterations, double l1_tolerance,
                  int dangling, double* ranks, uint32_t* iterations_run, int ptr_kind, void* stream) {
  return cmvg_pagerank_ex(g, degrees, alpha, iterations, l1_tolerance, dangling, nullptr, ranks, iterations_run,
                          ptr_kind, stream);
}

int cmvg_pagerank_step(cmvg_graph* g, const double* q, const uint32_t* deg, double alpha, double dmass, int dangling,
                       const double* p_prev, double* p_next, double* q_next, double* partial, void* stream) {
  return guarded([&] {
    require(g && q && deg && p_next && q_next && partial, "null argument");
    require(alpha > 0.0 && alpha < 1.0, "alpha must be in (0,1)");
    DeviceGuard dg(g->device);
    pagerank_step(g, q, deg, alpha, dmass, dangling, p_prev, p_next, q_next, partial, (cudaStream_t)stream);
  });
}

int cmvg_pagerank_step_push(cmvg_graph* g, const double* q, const uint32_t* deg, double alpha, double dmass,
                            int dangling, const double* p_prev, double* p_next, double* q_next, double* partial,
                            const uint8_t* push_mask, double* const* push_dst, void* stream) {
  return guarded([&] {
    require(g && q && deg && p_next && q_next && partial, "null argument");
    require(alpha > 0.0 && alpha < 1.0, "alpha must be in (0,1)");
    require((push_mask == nullptr) == (push_dst == nullptr), "push_mask and push_dst go together");
    DeviceGuard dg(g->device);
    pagerank_step(g, q, deg, alpha, dmass, dangling, p_prev, p_next, q_next, partial, (cudaStream_t)stream,
                  push_mask, push_dst);
  });
}

int cmvg_pagerank_step_dev(cmvg_graph* g, const double* q, const uint32_t* deg, double alpha, const double* dmass_dev,
                           int dangling, const double* p_prev, double* p_next, double* q_next, double* partial,
                           const uint8_t* push_mask, double* const* push_dst, void* stream) {
  return guarded([&] {
    require(g && q && deg && dmass_dev && p_next && q_next && partial, "null argument");
    require(alpha > 0.0 && alpha < 1.0, "alpha must be in (0,1)");
    require((push_mask == nullptr) == (push_dst == nullptr), "push_mask and push_dst go together");
    DeviceGuard dg(g->device);
    pagerank_step(g, q, deg, alpha, 0.0, dangling, p_prev, p_next, q_next, partial, (cudaStream_t)stream, push_mask,
                  push_dst, dmass_dev);
  });
}

}  // extern "C"
