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
