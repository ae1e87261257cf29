// bvf_matmat: Y = A X for X of shape n x k (row-major fp32, leading dimension
// ld) on the BV-F flat term layout (host/layout.hpp) -- BASELINE.json config
// 5, the multi-vector extension of the reference's product
// (ref_matvec.hpp:20-31), decoding amortised over KC = 4 columns per pass.
//
// The same block structure as the gather (cuda/bvf_gather.cuh), 256 threads
// per 1024-row block, with every table entry, term and row record carrying KC
// columns, in fp32 throughout (no fp32 -> fp64 conversions):
//   1. staging: each thread loads its 6 window rows (16 bytes of X each) and
//      the far slots; per column the block's largest exponent fixes an fp32
//      grid G_c = 2^(E_c - (cbits - 29)) (the transcoder's fp64 bound moved to
//      a 24-bit significand, less 2 bits of headroom for F), each value
//      splits exactly into h = (x + s) - s and l = x - h, and the window
//      prefix F = (sum h exact, sum l) is scanned per column;
//   2. terms: one 16-byte table load per term (x row or F hi row), +-split
//      into per-column (h, l) sums, F terms add their lo row (a predicated
//      16-byte load); a row end stores the row's 8 sums (32 bytes);
//   3. carries across chunk boundaries, reference chains, the 16-byte store of
//      each row's KC outputs.
// Sums of h are exact in fp32 (the transcoder bounds every partial sum), so
// the differential evaluation's cancellation costs nothing; the rounding left
// is that of the small l sums -- far inside the fp32 tolerance (1e-5).
#pragma once
#include <cstdint>

#include "bvf_gather.cuh"

namespace cmvg {

constexpr uint32_t kBmmCols = 4;          // columns per pass
constexpr uint32_t kBmmW = 1536, kBmmB = 1024, kBmmT = 256, kBmmXPer = kBmmW / kBmmT;
static_assert(kBmmB * 16u == 16384u, "the row-end store addresses the l plane at +16384");

struct BmmSmem {
  uint32_t off_tab, off_flo, off_rows, off_rn, off_misc, total;
};
// one table of 16-byte rows: x window, far slots, zero row, then F hi; F lo;
// row records as two planes of 16-byte rows, h[4] of every row then l[4]
// (consecutive rows in consecutive bank groups: a quarter warp's record loads
// of 8 consecutive rows are conflict-free; 32-byte records put rows p and
// p + 4 in the same banks)
__host__ __device__ constexpr BmmSmem bmm_smem_layout() {
  return BmmSmem{0u,
                 (bvf_f0(kBmmW) + kBmmW + 1) * 16u,
                 (bvf_f0(kBmmW) + kBmmW + 1) * 16u + (kBmmW + 1) * 16u,
                 (bvf_f0(kBmmW) + kBmmW + 1) * 16u + (kBmmW + 1) * 16u + kBmmB * 32u,
                 (bvf_f0(kBmmW) + kBmmW + 1) * 16u + (kBmmW + 1) * 16u + kBmmB * 32u + kBvfRnWords * 8u,
                 (bvf_f0(kBmmW) + kBmmW + 1) * 16u + (kBmmW + 1) * 16u + kBmmB * 32u + kBvfRnWords * 8u + 2048u};
}

struct BmmX {
  const float* X;   // column chunk base (X + c0)
  uint32_t ld, kk;  // leading dimension, columns of this chunk (<= 4)
  bool vec;         // 16-byte aligned rows and kk == 4: float4 loads
  __device__ __forceinline__ float4 row(uint32_t r) const {
    const float* p = X + (size_t)r * ld;
    if (vec) return __ldg(reinterpret_cast<const float4*>(p));
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (kk > 0) v.x = __ldg(p);
    if (kk > 1) v.y = __ldg(p + 1);
    if (kk > 2) v.z = __ldg(p + 2);
    if (kk > 3) v.w = __ldg(p + 3);
    return v;
  }
};

__device__ __forceinline__ float bmm_flip(float v, uint32_t sm) { return __int_as_float(__float_as_int(v) ^ (int)sm); }
__device__ __forceinline__ uint32_t bmm_exp(float v) { return ((uint32_t)__float_as_int(v) >> 23) & 0xffu; }

struct BmmAcc {
  float h[kBmmCols], l[kBmmCols];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (uint32_t c = 0; c < kBmmCols; ++c) h[c] = l[c] = 0.f;
  }
};

struct BmmTerms {
  uint32_t tab;   // shared address of the 16-byte table
  uint32_t flo;   // shared address of F lo minus F0 * 16
  uint32_t f0b;   // F0 * 16
  uint32_t rows;  // shared address of the row records
  float sg[kBmmCols];
  const float4* esc;  // x rows of this chunk's escape terms (bmm_esc_gather)
  // one term; END: the high term of a word (rows have an even term count)
  template <bool END, bool ESC>
  __device__ __forceinline__ void term(uint32_t c, uint32_t signw, BmmAcc& a, uint32_t& rowp) const {
    const uint32_t off = (c << 4) & (kBvfIdxMask << 4);
    const bool e = ESC && (c & kBvfEsc);
    float4 v;
    if (e) {
      v = __ldg(esc + (c & kBvfIdxMask));
    } else {
      asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(tab + off));
    }
    const uint32_t sm = signw & 0x80000000u;
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (uint32_t q = 0; q < kBmmCols; ++q) {
      const float xv = bmm_flip(x[q], sm);
      const float hv = (xv + sg[q]) - sg[q];
      a.h[q] += hv;
      a.l[q] += xv - hv;
    }
    {  // F term: its lo row (a predicated load, zeros otherwise; no branch)
      const uint32_t isf = (off >= f0b && !e) ? 1u : 0u;
      float4 w;
      asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %4, 0;\n\t"
          "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
          "@p ld.shared.v4.f32 {%0, %1, %2, %3}, [%5];\n\t}"
          : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w)
          : "r"(isf), "r"(flo + off));
      a.l[0] += bmm_flip(w.x, sm);
      a.l[1] += bmm_flip(w.y, sm);
      a.l[2] += bmm_flip(w.z, sm);
      a.l[3] += bmm_flip(w.w, sm);
    }
    if (END) {  // a row end: predicated stores of the row's sums, then restart
      const uint32_t end = c & kBvfEnd;
      const uint32_t p = rows + rowp * 16u;  // h plane; the l plane B x 16 bytes after it
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
                   "@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n\t"
                   "@p st.shared.v4.f32 [%1+16384], {%6, %7, %8, %9};\n\t}" ::"r"(end),
                   "r"(p), "f"(a.h[0]), "f"(a.h[1]), "f"(a.h[2]), "f"(a.h[3]), "f"(a.l[0]), "f"(a.l[1]), "f"(a.l[2]),
                   "f"(a.l[3]));
      rowp += end ? 1u : 0u;
#pragma unroll
      for (uint32_t q = 0; q < kBmmCols; ++q) {
        a.h[q] = end ? 0.f : a.h[q];
        a.l[q] = end ? 0.f : a.l[q];
      }
    }
  }
  template <bool ESC>
  __device__ __forceinline__ void word(uint32_t w, BmmAcc& a, uint32_t& rowp) const {
    term<false, ESC>(w & 0xffffu, w << 16, a, rowp);
    term<true, ESC>(w >> 16, w, a, rowp);
  }
};

// column chunk ch (grid y) of the X rows of a chunk: xs for columns [4 ch, 4 ch + 4)
__device__ __forceinline__ BmmX bmm_chunk(const float* X, uint32_t k, bool vec, uint32_t ch) {
  const uint32_t c0 = ch * kBmmCols;
  return BmmX{X + c0, k, min(kBmmCols, k - c0), vec && k - c0 >= kBmmCols};
}

// escape rows: xe[ch * cnt + i] = X[esc[i], 4 ch .. 4 ch + 4), chunk ch = blockIdx.y
__global__ void __launch_bounds__(256) bmm_esc_gather(const uint32_t* __restrict__ esc, uint64_t cnt,
                                                      const float* __restrict__ X, uint32_t k, bool vec,
                                                      float4* __restrict__ xe) {
  const BmmX xs = bmm_chunk(X, k, vec, blockIdx.y);
  xe += (size_t)blockIdx.y * cnt;
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += step) xe[i] = xs.row(__ldg(esc + i));
}

__global__ void __launch_bounds__(kBmmT, 2)
    bvf_matmat_kernel(BvfDev g, const float* __restrict__ X, uint32_t k, bool vec, uint32_t nch,
                      const float4* __restrict__ xe, uint64_t ne, float* __restrict__ Y) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr uint32_t W = kBmmW, B = kBmmB, T = kBmmT, E = kBmmXPer;
  constexpr BmmSmem L = bmm_smem_layout();
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  // the nch column chunks of a block are adjacent CTAs: they run together, so
  // the block's terms, X sectors and Y sectors are shared in L2 (one DRAM
  // read of each, whole-sector Y writes)
  const uint32_t chk = blockIdx.x % nch, bl = blockIdx.x / nch, b = g.block_begin + bl;
  const BmmX xs = bmm_chunk(X, k, vec, chk);
  xe += (size_t)chk * ne;
  Y += chk * kBmmCols;
  const uint32_t ldy = k;
  const BvfBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * B, nr = min(B, g.n - r0);
  const uint32_t* bs = g.words + bi.word_offset;
  const uint32_t nact = bi.nact, nslot = bi.nslot;
  const uint32_t F0 = bvf_f0(W);
  float4* tab = reinterpret_cast<float4*>(smem + L.off_tab);
  float4* flo = reinterpret_cast<float4*>(smem + L.off_flo);
  uint8_t* r8 = reinterpret_cast<uint8_t*>(smem + L.off_rn);
  float* miscf = reinterpret_cast<float*>(smem + L.off_misc);
  uint32_t* miscu = reinterpret_cast<uint32_t*>(smem + L.off_misc);
  const uint32_t rows_s = smem_u32(smem + L.off_rows);

  // ---- loads
  const bool active = tid < nact;
  const uint32_t* cw = bs + bi.codes_off + tid;
  if (tid == 32 && chk == 0) {
    const uint32_t cb = bi.nwords - bi.codes_off;
    if (cb > 8 * nact) bulk_prefetch_l2(bs + bi.codes_off + 8 * nact, ((cb - 8 * nact) * 4u) & ~15u);
    if (g.ahead && bl + g.ahead < g.nlaunch) asm volatile("prefetch.global.L2 [%0];" ::"l"(g.blocks + bl + g.ahead));
  }
  // half a wave ahead: the block whose CTA takes a slot next -- its header and
  // terms now, the X rows of its window after this block's terms (the
  // staging loads are the kernel's exposed latency)
  const bool pf = g.ahead && bl + g.ahead / 2 < g.nlaunch;
  const uint32_t pf_wlo = pf ? __ldg(&g.blocks[bl + g.ahead / 2].wlo) : 0u;
  if (tid == 64 && pf && chk == 0) {
    const BvfBlockInfo nb = g.blocks[bl + g.ahead / 2];
    if (nb.flags & kBvfFlagEsc) {
      bulk_prefetch_l2(g.words + nb.word_offset, nb.esc_off * 4u);
      bulk_prefetch_l2(g.words + nb.word_offset + nb.codes_off, (nb.nwords - nb.codes_off) * 4u);
    } else {
      bulk_prefetch_l2(g.words + nb.word_offset, nb.nwords * 4u);
    }
  }
  uint32_t w0[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w0[i] = active ? __ldg(cw + (size_t)i * nact) : 0u;
  const uint32_t srow = active ? (uint32_t)reinterpret_cast<const uint16_t*>(bs)[tid] : 0u;
  const uint32_t j0 = tid * E;
  float4 xv[E];
#pragma unroll
  for (uint32_t q = 0; q < E; ++q) {
    const uint32_t c = bi.wlo + j0 + q;
    xv[q] = c < g.n ? xs.row(c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float4 fv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid < nslot) fv = xs.row(__ldg(bs + bvf_far_off(nact) + tid));
  const uint32_t rnw = tid < kBvfRnWords ? __ldg(bs + bvf_rn_off(nact) + tid) : 0u;
  const float4* xeb = xe;
  uint32_t nesc = 0;
  if (bi.flags & kBvfFlagEsc) {
    xeb = xe + __ldg(g.esc_base + bl);
    nesc = __ldg(bs + bi.esc_off + nact);
  }

  // ---- per-column block exponents (non-finite: 0xff) -> grids
  uint32_t em[4] = {0, 0, 0, 0};
  auto see = [&](const float4& v) {
    em[0] = max(em[0], bmm_exp(v.x));
    em[1] = max(em[1], bmm_exp(v.y));
    em[2] = max(em[2], bmm_exp(v.z));
    em[3] = max(em[3], bmm_exp(v.w));
  };
#pragma unroll
  for (uint32_t q = 0; q < E; ++q) see(xv[q]);
  see(fv);
  for (uint32_t i = tid; i < nesc; i += T) see(__ldg(xeb + i));
#pragma unroll
  for (uint32_t q = 0; q < 4; ++q) em[q] = __reduce_max_sync(0xffffffffu, em[q]);
  if (lane < 4) miscu[warp * 4 + lane] = lane == 0 ? em[0] : lane == 1 ? em[1] : lane == 2 ? em[2] : em[3];
  __syncthreads();  // #1
  float sg[4];
  {
    // cbits - 27 would move the fp64 bound to 24 bits exactly; 2 more bits of
    // headroom keep F hi (up to W x 2^E) inside the split's exact range
    const int cb32 = max(1, (int)bi.cbits - 29);
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      uint32_t e = 0;
#pragma unroll
      for (uint32_t w = 0; w < T / 32; ++w) e = max(e, miscu[w * 4 + q]);
      // sigma = 1.5 * 2^(g + 23), g = E - cbits32, E = e - 127 + 1; 0 for non-finite or all-zero columns
      const int ef = (int)e + 1 + 23 - cb32;
      sg[q] = (e == 0xffu || e == 0u) ? 0.f : __int_as_float((max(ef, 1) << 23) | 0x400000);
    }
  }
  // ---- the x table rows (own window entries, far slots, the zero row)
  // a thread's rows are 6 x 16 bytes apart, so lanes 4..7 of each quarter warp
  // store theirs rotated by one row: the 8 lanes of a 16-byte store phase
  // then hit 8 different bank groups
  const bool rot = (tid >> 2) & 1u;
  static_assert(E == 6, "the store rotation assumes 6 rows per thread");
#pragma unroll
  for (uint32_t q = 0; q < E; ++q) tab[j0 + (rot ? (q + 1) % E : q)] = rot ? xv[(q + 1) % E] : xv[q];
  if (tid < nslot) tab[W + tid] = fv;
  if (tid == 0) tab[bvf_zero(W)] = make_float4(0.f, 0.f, 0.f, 0.f);
  // ---- window prefix per column: F hi = sum h (exact), F lo = sum l
  float sh[4] = {0.f, 0.f, 0.f, 0.f}, sl[4] = {0.f, 0.f, 0.f, 0.f};
  auto split = [&](float v, float s, float& h, float& l) {
    h = (v + s) - s;
    l = v - h;
  };
#pragma unroll
  for (uint32_t q = 0; q < E; ++q) {
    const float x4[4] = {xv[q].x, xv[q].y, xv[q].z, xv[q].w};
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
      float h, l;
      split(x4[c], sg[c], h, l);
      sh[c] += h;
      sl[c] += l;
    }
  }
  float ih[4], il[4];
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) {
    ih[c] = sh[c];
    il[c] = sl[c];
  }
#pragma unroll
  for (uint32_t o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
      const float uh = __shfl_up_sync(0xffffffffu, ih[c], o), ul = __shfl_up_sync(0xffffffffu, il[c], o);
      if (lane >= o) {
        ih[c] += uh;
        il[c] += ul;
      }
    }
  }
  if (lane == 31) {
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
      miscf[64 + warp * 8 + c] = ih[c];
      miscf[64 + warp * 8 + 4 + c] = il[c];
    }
  }
  __syncthreads();  // #2
  float bh[4], blo[4];
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) {
    bh[c] = ih[c] - sh[c];
    blo[c] = il[c] - sl[c];
  }
  for (uint32_t w = 0; w < warp; ++w) {
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
      bh[c] += miscf[64 + w * 8 + c];
      blo[c] += miscf[64 + w * 8 + 4 + c];
    }
  }
  float4* fhi = tab + F0;
  float4 fh[E], fl[E];
#pragma unroll
  for (uint32_t q = 0; q < E; ++q) {
    fh[q] = make_float4(bh[0], bh[1], bh[2], bh[3]);
    fl[q] = make_float4(blo[0], blo[1], blo[2], blo[3]);
    const float x4[4] = {xv[q].x, xv[q].y, xv[q].z, xv[q].w};
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
      float h, l;
      split(x4[c], sg[c], h, l);
      bh[c] += h;
      blo[c] += l;
    }
  }
#pragma unroll
  for (uint32_t q = 0; q < E; ++q) {
    fhi[j0 + (rot ? (q + 1) % E : q)] = rot ? fh[(q + 1) % E] : fh[q];
    flo[j0 + (rot ? (q + 1) % E : q)] = rot ? fl[(q + 1) % E] : fl[q];
  }
  if (tid == T - 1) {  // F[W]
    fhi[W] = make_float4(bh[0], bh[1], bh[2], bh[3]);
    flo[W] = make_float4(blo[0], blo[1], blo[2], blo[3]);
  }
  if (tid < kBvfRnWords) {  // r nibbles -> bytes
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      lo |= ((rnw >> (4 * q)) & 15u) << (8 * q);
      hi |= ((rnw >> (4 * q + 16)) & 15u) << (8 * q);
    }
    reinterpret_cast<uint2*>(r8)[tid] = make_uint2(lo, hi);
  }
  __syncthreads();  // #3

  // ---- terms
  BmmAcc acc;
  acc.zero();
  uint32_t rowp = srow;
  if (active) {
    BmmTerms tm;
    tm.tab = smem_u32(tab);
    tm.flo = smem_u32(flo) - F0 * 16u;
    tm.f0b = F0 * 16u;
    tm.rows = rows_s;
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) tm.sg[c] = sg[c];
    const bool esc = bi.flags & kBvfFlagEsc;
    tm.esc = esc ? xeb + __ldg(bs + bi.esc_off + tid) : xeb;
    const uint32_t nwords = bi.K / 2;
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = w0[i];
    for (uint32_t q = 8;; q += 8) {
      uint32_t nx[8];
      const bool more = q < nwords;
      if (more) {
#pragma unroll
        for (int i = 0; i < 8; ++i) nx[i] = __ldg(cw + (size_t)(q + i) * nact);
      }
      if (esc) {
#pragma unroll
        for (int i = 0; i < 8; ++i) tm.word<true>(w[i], acc, rowp);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) tm.word<false>(w[i], acc, rowp);
      }
      if (!more) break;
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = nx[i];
    }
  }
  if (pf) {
#pragma unroll
    for (uint32_t q = 0; q < E; ++q) {
      const uint32_t c = pf_wlo + q * T + tid;
      if (c < g.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(xs.X + (size_t)c * xs.ld));
    }
  }
  // ---- carries: rows cut by chunk boundaries get the tails of the chunks before
  // their end (segmented scan of the 8 tail sums, in the warp then across warps)
  const bool has_end = active && rowp != srow;
  float t8[8];
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) {
    t8[c] = acc.h[c];
    t8[4 + c] = acc.l[c];
  }
  bool sf = has_end;
  if (!__all_sync(0xffffffffu, has_end || !active)) {
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      float u[8];
#pragma unroll
      for (uint32_t c = 0; c < 8; ++c) u[c] = __shfl_up_sync(0xffffffffu, t8[c], o);
      const bool uf = __shfl_up_sync(0xffffffffu, sf, o);
      if (lane >= o) {
        if (!sf) {
#pragma unroll
          for (uint32_t c = 0; c < 8; ++c) t8[c] += u[c];
        }
        sf = sf || uf;
      }
    }
  }
  if (lane == 31) {
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) miscf[128 + warp * 8 + c] = t8[c];
    miscu[32 + warp] = sf;
  }
  float ch[8];
#pragma unroll
  for (uint32_t c = 0; c < 8; ++c) ch[c] = __shfl_up_sync(0xffffffffu, t8[c], 1);
  const bool cf = __shfl_up_sync(0xffffffffu, sf, 1);
  if (lane == 0) {
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) ch[c] = 0.f;
  }
  __syncthreads();  // #4
  if (has_end) {
    if (lane == 0 || !cf) {
      for (int w = (int)warp - 1; w >= 0; --w) {
#pragma unroll
        for (uint32_t c = 0; c < 8; ++c) ch[c] += miscf[128 + w * 8 + c];
        if (miscu[32 + w]) break;
      }
    }
    float4* rr = reinterpret_cast<float4*>(smem + L.off_rows) + srow;
    float4 a = rr[0], c2 = rr[B];
    a.x += ch[0];
    a.y += ch[1];
    a.z += ch[2];
    a.w += ch[3];
    c2.x += ch[4];
    c2.y += ch[5];
    c2.z += ch[6];
    c2.w += ch[7];
    rr[0] = a;
    rr[B] = c2;
  }
  __syncthreads();  // #5

  // ---- reference chains and the stores
  const float4* rec = reinterpret_cast<const float4*>(smem + L.off_rows);
  float* yb = Y + (size_t)(r0 - g.row_begin) * ldy;
  const bool yvec = xs.vec && (ldy % 4u) == 0 && ((reinterpret_cast<uintptr_t>(Y) & 15u) == 0);
  auto store = [&](uint32_t k, const float4& h, const float4& l) {
    const float4 y = make_float4(h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w);
    float* p = yb + (size_t)k * ldy;
    if (yvec) {
      *reinterpret_cast<float4*>(p) = y;
    } else {
      if (xs.kk > 0) p[0] = y.x;
      if (xs.kk > 1) p[1] = y.y;
      if (xs.kk > 2) p[2] = y.z;
      if (xs.kk > 3) p[3] = y.w;
    }
  };
  auto add4 = [](float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
  };
  if (g.max_depth <= 3) {
    for (uint32_t k = tid; k < nr; k += T) {
      float4 h = rec[k], l = rec[B + k];
      uint32_t p = k, r = r8[k];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if (r) {
          p -= r;
          add4(h, rec[p]);
          add4(l, rec[B + p]);
          r = r8[p];
        }
      }
      store(k, h, l);
    }
  } else {
    // unbounded chains: pointer jumping, one barrier-separated level per step
    // (the table region is dead after the terms)
    constexpr uint32_t kMaxPer = B / T;
    constexpr uint16_t kNone = 0xffffu;
    uint16_t* ptr = reinterpret_cast<uint16_t*>(smem + L.off_tab);
    float4* rw = reinterpret_cast<float4*>(smem + L.off_rows);
    int any = 0;
    for (uint32_t k = tid; k < nr; k += T) {
      const uint32_t r = r8[k];
      ptr[k] = r ? (uint16_t)(k - r) : kNone;
      any |= (r != 0);
    }
    any = __syncthreads_or(any);
    while (any) {
      float4 nh[kMaxPer], nl[kMaxPer];
      uint16_t np_[kMaxPer];
      int more = 0;
#pragma unroll
      for (uint32_t q = 0; q < kMaxPer; ++q) {
        const uint32_t k = tid + q * T;
        if (k < nr) {
          const uint32_t p = ptr[k];
          float4 h = rw[k], l = rw[B + k];
          uint16_t pn = kNone;
          if (p != kNone) {
            add4(h, rw[p]);
            add4(l, rw[B + p]);
            pn = ptr[p];
          }
          nh[q] = h;
          nl[q] = l;
          np_[q] = pn;
          more |= (pn != kNone);
        }
      }
      __syncthreads();
#pragma unroll
      for (uint32_t q = 0; q < kMaxPer; ++q) {
        const uint32_t k = tid + q * T;
        if (k < nr) {
          rw[k] = nh[q];
          rw[B + k] = nl[q];
          ptr[k] = np_[q];
        }
      }
      any = __syncthreads_or(more);
    }
    for (uint32_t k = tid; k < nr; k += T) store(k, rw[k], rw[B + k]);
  }
}

}  // namespace cmvg
