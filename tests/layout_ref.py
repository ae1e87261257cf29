"""Python re-implementation of the device kernels' view of the BV-D layout
(host/layout.hpp): row bit offsets from the headers, the escape table, and the
per-row code decode.  The CPU tests use it to check that the layout builder's
output reproduces the adjacency exactly -- the same arithmetic the sm_100a
kernels perform (cuda/bvd_common.cuh row_setup, cuda/bvd_gather.cuh)."""
import numpy as np

MINUS_ESC, RES_ESC, INT_ESC = 31, 63, 15


def hdr_fields(h):
    h = int(h)
    return dict(r=h >> 29, nm=(h >> 24) & 31, ns=(h >> 18) & 63, ni=(h >> 14) & 15, wp=(h >> 9) & 31,
                wl=(h >> 4) & 31, far=(h >> 3) & 1)


def bias(wp):
    return (1 << (wp - 1)) if wp else 0


def extract(words, off, w):
    if w == 0:
        return 0
    wi, sh = off >> 5, off & 31
    win = ((int(words[wi]) << 32) | int(words[wi + 1])) << sh
    win &= (1 << 64) - 1
    return win >> (64 - w)


def unfold(u):
    return -((u + 1) >> 1) if (u & 1) else (u >> 1)


def decode_layout(words, blocks, n, B, lmin, W=None):
    """Returns (refs, rows) per row: (ref distance, sorted adjacency).  With the
    window size W, also checks the `far` flag against the block's x-window."""
    rows_out = [None] * n
    refs_out = [0] * n
    for b in range(len(blocks)):
        woff = int(blocks[b, 0]) | (int(blocks[b, 1]) << 32)
        nw = int(blocks[b, 2])
        base = words[woff:woff + nw + 8]
        r0 = b * B
        nr = min(B, n - r0)
        hdrs = [hdr_fields(base[k]) for k in range(nr)]
        escaped = [h["nm"] == MINUS_ESC or h["ns"] == RES_ESC or h["ni"] == INT_ESC for h in hdrs]
        nesc = sum(escaped)
        assert nesc == int(blocks[b, 4])
        esc = {int(base[B + 4 * e]): (int(base[B + 4 * e + 1]), int(base[B + 4 * e + 2]), int(base[B + 4 * e + 3]))
               for e in range(nesc)}
        off = (B + 4 * nesc) * 32
        for k in range(nr):
            h = hdrs[k]
            nm, ns, ni = esc[k] if escaped[k] else (h["nm"], h["ns"], h["ni"])
            wp, wl, r = h["wp"], h["wl"], h["r"]
            i = r0 + k
            ib = i - bias(wp)
            pts = []
            for t in range(nm + ns):
                pts.append(ib + extract(base, off, wp))
                off += wp
            ints = []
            for t in range(ni):
                left = ib + extract(base, off, wp)
                ln = extract(base, off + wp, wl) + lmin
                ints.append((left, ln))
                off += wp + wl
            minus, res = pts[:nm], pts[nm:]
            if W is not None:
                wlo = int(blocks[b, 3])
                far = any(not (wlo <= c < wlo + W) for c in pts) or any(
                    not (wlo <= left and left + ln <= wlo + W) for left, ln in ints)
                assert bool(h["far"]) == far, (i, h, far)
            plus = set(res)
            for left, ln in ints:
                plus.update(range(left, left + ln))
            if r:
                assert k >= r, "reference crosses a block"
                row = (set(rows_out[i - r]) - set(minus)) | plus
            else:
                assert not minus
                row = plus
            rows_out[i] = sorted(row)
            refs_out[i] = r
    return refs_out, rows_out


# ---------------------------------------------------------------------------
# BV-S (sliced layout; host/layout.hpp, cuda/bvs_gather.cuh)
UNIT_PTS, UNIT_INTS, BIAS16 = 16, 2, 32768


def decode_sliced(words, blocks, n, B, lmin, W):
    """Decode the BV-S layout as the gather kernel reads it: heavy rows from the
    row-major bit stream, units from the lane-interleaved slice bodies; in
    multi slices a row's units occupy adjacent lanes starting at its primary.
    Returns (refs, rows) like decode_layout and checks the structural
    invariants (every row exactly one primary unit, slice metadata = max over
    lanes, class/far flags consistent, units within their limits)."""
    rows_out = [None] * n
    refs_out = [0] * n
    heavy_items = 0
    for b in range(len(blocks)):
        woff = int(blocks[b, 0]) | (int(blocks[b, 1]) << 32)
        nw = int(blocks[b, 2])
        wlo = int(blocks[b, 3])
        s = [int(v) for v in words[woff:woff + nw + 64]]
        r0 = b * B
        nr = min(B, n - r0)
        nsl, nh = s[0] & 0xFFFF, s[0] >> 16
        htab, hstr = s[1], s[2]
        assert s[3] == heavy_items  # the block's first heavy work item (global numbering)
        # static warp schedule: u16 table starts of the 8 warps, then the table size
        starts = [(s[4 + q // 2] >> (16 * (q % 2))) & 0xFFFF for q in range(9)]
        assert starts[0] == 0 and starts[8] == nsl and all(a <= b for a, b in zip(starts, starts[1:]))
        parts = {}   # k -> dict(minus, res, ints, r)

        def inwin(c):
            return wlo <= c < wlo + W
        item0 = 0
        for q in range(nh):
            e = htab + 6 * q
            sa, nm, ns, ni, boff = s[e], s[e + 1], s[e + 2], s[e + 3], s[e + 4]
            assert s[e + 5] == item0
            item0 += max(1, -(-(nm + ns) // 512))
            k, r, wp, wl = sa & 4095, (sa >> 12) & 7, (sa >> 15) & 31, (sa >> 20) & 31
            off = hstr * 32 + boff
            ib = r0 + k - bias(wp)
            pts = []
            for t in range(nm + ns):
                pts.append(ib + extract(s, off, wp))
                off += wp
            ints = []
            for t in range(ni):
                ints.append((ib + extract(s, off, wp), extract(s, off + wp, wl) + lmin))
                off += wp + wl
            assert k not in parts
            parts[k] = dict(minus=pts[:nm], res=pts[nm:], ints=ints, r=r)
        heavy_items += item0
        for sl in range(nsl):
            rec = s[10 + 2 * sl]
            meta = s[rec]
            assert s[10 + 2 * sl + 1] == meta
            mnp, mni, c32, far, multi = meta & 31, (meta >> 5) & 7, (meta >> 8) & 1, (meta >> 9) & 1, (meta >> 10) & 1
            rounds = (meta >> 11) & 7
            seen_np, seen_ni = 0, 0
            cur = None
            run, max_run = 0, 0  # units of the current row, most units of one row
            for lane in range(32):
                h = s[rec + 1 + lane]
                if not h >> 31:
                    cur = None
                    run = 0
                    continue
                prim, k, r = (h >> 30) & 1, (h >> 20) & 1023, (h >> 17) & 7
                nm, npt, ni = (h >> 12) & 31, (h >> 7) & 31, (h >> 4) & 7
                assert npt <= UNIT_PTS and ni <= UNIT_INTS and nm <= npt
                seen_np, seen_ni = max(seen_np, npt), max(seen_ni, ni)
                body = rec + 33 + lane
                lw = lambda q: s[body + 32 * q]  # noqa: E731
                pts, ints = [], []
                if not c32 and not far:
                    # near class 16: rectangular, padded window indices, sign in bit 15
                    zc = W + (W >> 3)
                    mnpw = (mnp + 1) >> 1
                    minus, res = [], []
                    for q in range(mnpw):
                        w = lw(q)
                        for c in (w >> 16, w & 0xFFFF):
                            if c == zc:
                                continue
                            pi = c & 0x7FFF
                            assert pi % 9 != 8
                            col = wlo + (pi // 9) * 8 + pi % 9
                            (minus if c >> 15 else res).append(col)
                    assert (len(minus), len(minus) + len(res)) == (nm, npt), (b, sl, lane)
                    pts = minus + res
                    for u in range(mni):
                        w = lw(mnpw + u)
                        if w:
                            ints.append((wlo + (w >> 16), w & 0xFFFF))
                    assert len(ints) == ni
                elif not c32:
                    for t in range(npt):
                        w = lw(t >> 1)
                        pts.append(wlo - BIAS16 + ((w & 0xFFFF) if t & 1 else (w >> 16)))
                    q0 = (npt + 1) >> 1
                    for u in range(ni):
                        w = lw(q0 + u)
                        ints.append((wlo - BIAS16 + (w >> 16), (w & 0xFFFF) + lmin))
                else:
                    pts = [lw(t) for t in range(npt)]
                    for u in range(ni):
                        ints.append((lw(npt + 2 * u), lw(npt + 2 * u + 1) + lmin))
                ufar = any(not inwin(c) for c in pts) or any(
                    not (inwin(a) and inwin(a + ln - 1)) for a, ln in ints)
                if not far:
                    assert not ufar, (b, sl, lane)
                run = 1 if prim else run + 1
                max_run = max(max_run, run)
                if prim:
                    assert k not in parts
                    cur = k
                    parts[k] = dict(minus=pts[:nm], res=pts[nm:], ints=ints, r=r)
                else:
                    assert multi and cur is not None, (b, sl, lane)
                    assert k == 0 and r == 0
                    parts[cur]["minus"] += pts[:nm]
                    parts[cur]["res"] += pts[nm:]
                    parts[cur]["ints"] += ints
            assert (seen_np, seen_ni) == (mnp, mni), (b, sl)
            # the segmented reduction's rounds cover the longest row: 2^rounds >= units
            assert (1 << rounds) >= max_run and (rounds == 0 or (1 << (rounds - 1)) < max_run), (b, sl, rounds, max_run)
        assert sorted(parts) == list(range(nr))
        for k in range(nr):
            p = parts[k]
            i = r0 + k
            plus = set(p["res"])
            for left, ln in p["ints"]:
                plus.update(range(left, left + ln))
            if p["r"]:
                assert k >= p["r"]
                row = (set(rows_out[i - p["r"]]) - set(p["minus"])) | plus
            else:
                assert not p["minus"]
                row = plus
            rows_out[i] = sorted(row)
            refs_out[i] = p["r"]
    return refs_out, rows_out


# ---------------------------------------------------------------------------
# BV-T (target-sorted scatter layout; host/layout.hpp, cuda/bvt_scatter.cuh)
def scatter_bvt_int(words, blocks, n, B, W, x):
    """y = x A evaluated from the BV-T layout exactly as the two scatter kernels
    do, in integer arithmetic (x integer): coefficients c_k from the ref table,
    per-target segmented sums of the 16-bit codes, inclusive prefix of the
    difference targets, far slots, then the window combine.  Also checks the
    structural invariants (one primary per target, slice metadata)."""
    x = np.asarray(x, dtype=np.int64)
    y = np.zeros(n, dtype=np.int64)
    for b in range(len(blocks)):
        woff = int(blocks[b, 0]) | (int(blocks[b, 1]) << 32)
        nw = int(blocks[b, 2])
        wlo = int(blocks[b, 3])
        s = [int(v) for v in words[woff:woff + nw + 64]]
        r0 = b * B
        nr = min(B, n - r0)
        nsl, nh = s[0] & 0xFFFF, s[0] >> 16
        htab, hcode, nfar, cs, fl = s[1], s[2], s[3], s[4], s[5]
        c = [int(x[r0 + k]) for k in range(nr)] + [0] * (B + 1 - nr)
        nlev = s[cs]
        starts = s[cs + 1:cs + nlev + 2]
        ent = cs + nlev + 2
        for lv in range(nlev):  # deepest level first; rows pull their children
            for i in range(starts[lv], starts[lv + 1]):
                e = s[ent + i]
                k, m = e & 1023, e >> 10
                for r in range(1, 8):
                    if m >> (r - 1) & 1:
                        c[k] += c[k + r]
        far_cols = s[fl:fl + nfar]
        assert far_cols == sorted(far_cols) and len(set(far_cols)) == nfar
        assert all(not (wlo <= col < wlo + W) for col in far_cols)
        out = {}

        def term(code):
            return -c[code & 0x7FFF] if code >> 15 else c[code & 0x7FFF]
        for q in range(nh):
            t, ne, co = s[htab + 3 * q], s[htab + 3 * q + 1], hcode + s[htab + 3 * q + 2]
            assert ne > 512 and t not in out
            tot = 0
            for i in range(ne):
                w = s[co + i // 2]
                tot += term((w & 0xFFFF) if i & 1 else (w >> 16))
            out[t] = tot
        cur = None
        for sl in range(nsl):
            rec = s[8 + 2 * sl]
            meta = s[rec]
            assert s[8 + 2 * sl + 1] == meta
            mne, multi, rounds = meta & 1023, (meta >> 10) & 1, (meta >> 11) & 7
            mnw = (mne + 1) >> 1
            run, max_run = 0, 0  # units of the current target, most units of one target
            for lane in range(32):
                h = s[rec + 1 + lane]
                if not h >> 31:
                    run = 0
                    continue
                prim, t = (h >> 30) & 1, h & 0x3FFFFFFF
                run = 1 if prim else run + 1
                max_run = max(max_run, run)
                tot = 0
                for q in range(mnw):
                    w = s[rec + 33 + lane + 32 * q]
                    tot += term(w >> 16) + term(w & 0xFFFF)
                if prim:
                    assert t not in out
                    out[t] = tot
                    cur = t
                else:
                    assert multi and t == cur
                    out[cur] += tot
            assert (1 << rounds) >= max_run and (rounds == 0 or (1 << (rounds - 1)) < max_run)
        run = 0
        for j in range(W):
            run += out.get(W + j, 0)
            if wlo + j < n:
                y[wlo + j] += out.get(j, 0) + run
        for f, col in enumerate(far_cols):
            y[col] += out.get(2 * W + f, 0)
    return y


# ---------------------------------------------------------------------------
# BV-F (flat term stream; host/layout.hpp, cuda/bvf_gather.cuh)
BVF_SLOTS, BVF_IDX, BVF_ESC, BVF_END, BVF_MINUS, BVF_FLAG_ESC = 127, 0x1FFF, 0x2000, 0x4000, 0x8000, 1


def _align4(v):
    return (v + 3) & ~3


def bvf_block(words, blk):
    """Fields of one BV-F block: info dict, start rows, r per row, slot columns,
    escape starts and columns, and the terms of each chunk (list of lists)."""
    woff = int(blk[0]) | (int(blk[1]) << 32)
    info = dict(wlo=int(blk[2]), K=int(blk[3]) & 0xFFFF, nact=int(blk[3]) >> 16, nslot=int(blk[4]) & 0xFFFF,
                cbits=(int(blk[4]) >> 16) & 0xFF, flags=int(blk[4]) >> 24, codes_off=int(blk[5]),
                esc_off=int(blk[6]), nwords=int(blk[7]))
    s = words[woff:woff + info["nwords"]]
    nact, K = info["nact"], info["K"]
    sr = s[:(nact + 1) // 2].view(np.uint16)[:nact].astype(np.int64) if nact else np.zeros(0, np.int64)
    rn_off = _align4((nact + 1) // 2)
    rn = s[rn_off:rn_off + 128]
    r = np.array([(int(rn[k >> 3]) >> (4 * (k & 7))) & 15 for k in range(1024)], np.int64)
    far_off = rn_off + 128
    slots = s[far_off:far_off + info["nslot"]].astype(np.int64)
    escstart, esccol = None, None
    if info["flags"] & BVF_FLAG_ESC:
        eo = info["esc_off"]
        escstart = s[eo:eo + nact + 1].astype(np.int64)
        c0 = eo + _align4(nact + 1)
        esccol = s[c0:c0 + int(escstart[nact])].astype(np.int64)
    co = info["codes_off"]
    cw = s[co:co + (K // 2) * nact].reshape(K // 2, nact)  # word q of chunk t at [q, t]
    chunks = []
    for t in range(nact):
        wt = cw[:, t]
        codes = np.empty(K, np.int64)
        codes[0::2] = wt & 0xFFFF
        codes[1::2] = wt >> 16
        chunks.append(codes)
    return info, sr, r, slots, escstart, esccol, chunks


def gather_bvf(words, blocks, n, B, W, x, max_depth=3):
    """y = A x with the BV-F kernel's arithmetic (exact split at the block grid,
    chunk sums with row ends, carries, reference chains) in fp64."""
    x = np.asarray(x, np.float64)
    y = np.zeros(n)
    F0, ZERO = W + BVF_SLOTS + 1, W + BVF_SLOTS
    for b in range(len(blocks)):
        info, sr, r, slots, escstart, esccol, chunks = bvf_block(words, blocks[b])
        r0, nr, wlo = b * B, min(B, n - b * B), info["wlo"]
        tab = np.zeros(F0 + W + 1)
        flo = np.zeros(W + 1)
        win = np.zeros(W)
        hi_c = min(n, wlo + W)
        if hi_c > wlo:
            win[:hi_c - wlo] = x[wlo:hi_c]
        tab[:W] = win
        tab[W:W + len(slots)] = x[slots]
        vals = np.concatenate([win, x[slots]] + ([x[esccol]] if esccol is not None else []))
        fin = vals[np.isfinite(vals)]
        nonfin = len(fin) != len(vals)
        em = int(np.max((fin.view(np.uint64) >> np.uint64(52)) & np.uint64(0x7FF))) if len(fin) else 0
        sigma = 0.0
        if not nonfin:
            ef = max(em + 1 + 52 - info["cbits"], 1)
            sigma = float(np.array([(ef << 52) | (1 << 51)], np.uint64).view(np.float64)[0])
        sh = sl = 0.0
        for j in range(W):
            tab[F0 + j], flo[j] = sh, sl
            h = (win[j] + sigma) - sigma
            sh += h
            sl += win[j] - h
        tab[F0 + W], flo[W] = sh, sl
        rows = np.zeros((B, 2))
        tails, has_end = [], []
        for t, codes in enumerate(chunks):
            ah = al = 0.0
            row = int(sr[t])
            for c in codes:
                c = int(c)
                idx = c & BVF_IDX
                if c & BVF_ESC:
                    v = x[esccol[escstart[t] + idx]]
                    wl = 0.0
                else:
                    v = tab[idx]
                    wl = flo[idx - F0] if idx >= F0 else 0.0
                if c & BVF_MINUS:
                    v, wl = -v, -wl
                h = (v + sigma) - sigma
                ah += h
                al += (v - h) + wl
                if c & BVF_END:
                    rows[row] = (ah, al)
                    ah = al = 0.0
                    row += 1
            tails.append((ah, al))
            has_end.append(row > int(sr[t]))
        for t in range(1, len(chunks)):
            if not has_end[t]:
                continue
            ch = cl = 0.0
            j = t - 1
            while True:
                ch += tails[j][0]
                cl += tails[j][1]
                if j == 0 or has_end[j]:
                    break
                j -= 1
            rows[int(sr[t])] += (ch, cl)
        if max_depth <= 3:
            for k in range(nr):
                s_h, s_l = rows[k]
                p, rr = k, r[k]
                for _ in range(3):
                    if rr:
                        p -= rr
                        s_h += rows[p][0]
                        s_l += rows[p][1]
                        rr = r[p]
                y[r0 + k] = s_h + s_l
        else:
            vals2 = rows[:nr].copy()
            ptr = [k - r[k] if r[k] else -1 for k in range(nr)]
            while any(p >= 0 for p in ptr):
                nv, np_ = vals2.copy(), list(ptr)
                for k in range(nr):
                    if ptr[k] >= 0:
                        nv[k] += vals2[ptr[k]]
                        np_[k] = ptr[ptr[k]]
                vals2, ptr = nv, np_
            y[r0:r0 + nr] = vals2[:, 0] + vals2[:, 1]
    return y
