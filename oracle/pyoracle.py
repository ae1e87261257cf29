"""TEST INFRASTRUCTURE ONLY: ctypes wrapper over oracle/_build/libcmv_oracle.so,
the CPU restatement of the reference API (see cmv_oracle.hpp).  Imported only by
tests/, __graft_entry__.smoke() and bench.py's CPU legs -- never by the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "libcmv_oracle.so")
_lib = None
_P = C.c_void_p

NO_REF = 0xFFFFFFFF


def build() -> str:
    subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = C.CDLL(_LIB)
        sig = {
            "oracle_last_error": (C.c_char_p, []),
            "oracle_hw_threads": (C.c_uint, []),
            "oracle_csr_new": (_P, [C.c_uint32, _P, _P]),
            "oracle_build_csr": (_P, [_P, C.c_uint64, C.c_uint32]),
            "oracle_transpose": (_P, [_P]),
            "oracle_csr_n": (C.c_uint32, [_P]),
            "oracle_csr_m": (C.c_uint64, [_P]),
            "oracle_csr_offsets": (_P, [_P]),
            "oracle_csr_cols": (_P, [_P]),
            "oracle_csr_free": (None, [_P]),
            "oracle_out_degrees": (C.c_int, [_P, _P]),
            "oracle_matvec_csr": (C.c_int, [_P, _P, _P, C.c_uint]),
            "oracle_matvec_csr_raw": (C.c_int, [C.c_uint32, _P, _P, _P, _P, C.c_uint]),
            "oracle_compress": (_P, [_P, C.c_uint32, C.c_uint]),
            "oracle_rm_free": (None, [_P]),
            "oracle_rm_validate": (C.c_int, [_P]),
            "oracle_rm_arrays": (C.c_int, [_P] + [C.POINTER(_P)] * 5 + [C.POINTER(C.c_uint64)] * 2),
            "oracle_rm_new": (_P, [C.c_uint32, _P, _P, _P, _P, _P]),
            "oracle_stats": (C.c_int, [_P, _P, _P, C.POINTER(C.c_double)]),
            "oracle_reconstruct_row": (C.c_int, [_P, C.c_uint32, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
            "oracle_reconstruct_graph": (_P, [_P]),
            "oracle_matvec_ref": (C.c_int, [_P, _P, _P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
            "oracle_matvec_ref_concurrent": (C.c_double, [_P, _P, _P, C.c_uint]),
            "oracle_pagerank_csr": (C.c_int, [_P, _P, C.c_double, C.c_uint32, C.c_double, C.c_int, _P, _P,
                                              C.POINTER(C.c_uint32), C.c_uint]),
            "oracle_pagerank_ref": (C.c_int, [_P, _P, C.c_double, C.c_uint32, C.c_double, C.c_int, _P, _P,
                                              C.POINTER(C.c_uint32)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def _chk(rc):
    if rc == 0:
        return
    msg = lib().oracle_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise IndexError(msg)
    raise RuntimeError(msg)


def _ptr(a):
    return a.ctypes.data if a.size else None


def _view(ptr, count, dtype):
    if count == 0:
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (count * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count)


def threads() -> int:
    return int(lib().oracle_hw_threads())


class Csr:
    """cmv::CsrGraph (csr.hpp:16-36)."""

    def __init__(self, h):
        if not h:
            _chk(8)
        self.h = _P(h)
        self.n = int(lib().oracle_csr_n(self.h))
        self.m = int(lib().oracle_csr_m(self.h))

    @classmethod
    def from_arrays(cls, n, row_offsets, cols):
        ro = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        co = np.ascontiguousarray(cols, dtype=np.uint32)
        return cls(lib().oracle_csr_new(n, _ptr(ro), _ptr(co)))

    @classmethod
    def build(cls, edges, n):
        """cmv::build_csr (csr.hpp:41)."""
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        h = lib().oracle_build_csr(_ptr(e), len(e), n)
        if not h:
            _chk(2 if "endpoint" in lib().oracle_last_error().decode() else 8)
        return cls(h)

    @property
    def row_offsets(self):
        return _view(lib().oracle_csr_offsets(self.h), self.n + 1, np.uint64)

    @property
    def cols(self):
        return _view(lib().oracle_csr_cols(self.h) or 0, self.m, np.uint32)

    def row(self, u):
        ro = self.row_offsets
        return self.cols[int(ro[u]):int(ro[u + 1])]

    def transpose(self):
        return Csr(lib().oracle_transpose(self.h))

    def out_degrees(self):
        d = np.empty(self.n, dtype=np.uint32)
        _chk(lib().oracle_out_degrees(self.h, _ptr(d)))
        return d

    def matvec(self, x, nthreads=1):
        """cmv::matvec_csr (csr.hpp:51)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if len(x) != self.n:
            raise ValueError("matvec_csr: dimension mismatch")
        y = np.empty(self.n, dtype=np.float64)
        _chk(lib().oracle_matvec_csr(self.h, _ptr(x), _ptr(y), nthreads))
        return y

    def __del__(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.oracle_csr_free(self.h)
            self.h = None


def matvec_csr_raw(n, row_offsets, cols, x, nthreads=1):
    """matvec_csr over borrowed arrays (no graph copy)."""
    y = np.empty(n, dtype=np.float64)
    _chk(lib().oracle_matvec_csr_raw(n, _ptr(row_offsets), _ptr(cols), _ptr(x), _ptr(y), nthreads))
    return y


class RefMatrix:
    """cmv::ReferencedMatrix (ref_matrix.hpp:28-52)."""

    def __init__(self, h, n):
        if not h:
            _chk(1)
        self.h = _P(h)
        self.n = n

    @classmethod
    def compress(cls, g: Csr, window: int, nthreads: int = 1):
        """cmv::compress (ref_matrix.hpp:69)."""
        h = lib().oracle_compress(g.h, window, nthreads)
        if not h:
            _chk(1)
        return cls(h, g.n)

    @classmethod
    def from_arrays(cls, n, refs, plus_rows, minus_rows):
        refs = np.asarray([NO_REF if r is None else r for r in refs], dtype=np.uint32)
        po = np.zeros(n + 1, dtype=np.uint64)
        mo = np.zeros(n + 1, dtype=np.uint64)
        po[1:] = np.cumsum([len(r) for r in plus_rows])
        mo[1:] = np.cumsum([len(r) for r in minus_rows])
        pc = np.asarray([c for r in plus_rows for c in r] or [0], dtype=np.uint32)
        mc = np.asarray([c for r in minus_rows for c in r] or [0], dtype=np.uint32)
        return cls(lib().oracle_rm_new(n, _ptr(refs), _ptr(po), _ptr(pc), _ptr(mo), _ptr(mc)), n)

    def arrays(self):
        ptrs = [_P() for _ in range(5)]
        np_, nm = C.c_uint64(), C.c_uint64()
        lib().oracle_rm_arrays(self.h, *[C.byref(p) for p in ptrs], C.byref(np_), C.byref(nm))
        n = self.n
        refs = _view(ptrs[0].value, n, np.uint32)
        po = _view(ptrs[1].value, n + 1, np.uint64)
        pc = _view(ptrs[2].value or 0, np_.value, np.uint32)
        mo = _view(ptrs[3].value, n + 1, np.uint64)
        mc = _view(ptrs[4].value or 0, nm.value, np.uint32)
        return refs, po, pc, mo, mc

    def validate(self):
        _chk(lib().oracle_rm_validate(self.h))

    def stats(self, g: Csr):
        out = np.zeros(6, dtype=np.uint64)
        ratio = C.c_double()
        _chk(lib().oracle_stats(self.h, g.h, _ptr(out), C.byref(ratio)))
        return {"n": int(out[0]), "m": int(out[1]), "m_prime": int(out[2]), "rows_self_coded": int(out[3]),
                "max_chain": int(out[4]), "ratio_by_convention": bool(out[5]), "ratio": ratio.value}

    def reconstruct_row(self, i):
        cap = 1 << 20
        out = np.empty(cap, dtype=np.uint32)
        ln = C.c_uint64()
        _chk(lib().oracle_reconstruct_row(self.h, i, _ptr(out), cap, C.byref(ln)))
        return out[: ln.value].copy()

    def reconstruct_graph(self):
        return Csr(lib().oracle_reconstruct_graph(self.h))

    def matvec(self, x):
        """cmv::matvec_ref (ref_matvec.hpp:34-35) -> (y, (adds, references_used))."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(len(x), dtype=np.float64)
        adds, refs = C.c_uint64(), C.c_uint64()
        _chk(lib().oracle_matvec_ref(self.h, _ptr(x), _ptr(y), C.byref(adds), C.byref(refs)))
        return y, (adds.value, refs.value)

    def matvec_concurrent(self, x, nthreads):
        """nthreads independent products; returns wall seconds."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        ys = np.empty(len(x) * nthreads, dtype=np.float64)
        return float(lib().oracle_matvec_ref_concurrent(self.h, _ptr(x), _ptr(ys), nthreads))

    def __del__(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.oracle_rm_free(self.h)
            self.h = None


def pagerank_csr(at: Csr, degrees, alpha=0.15, iterations=10, l1_tolerance=None, dangling="uniform", start=None,
                 nthreads=1):
    """cmv::pagerank with CsrKernel(A^T) (pagerank.hpp:36-46,100-102)."""
    deg = np.ascontiguousarray(degrees, dtype=np.uint32)
    out = np.empty(at.n, dtype=np.float64)
    it = C.c_uint32()
    st = None if start is None else np.ascontiguousarray(start, dtype=np.float64)
    _chk(lib().oracle_pagerank_csr(at.h, _ptr(deg), alpha, iterations, -1.0 if l1_tolerance is None else l1_tolerance,
                                   0 if dangling == "uniform" else 1, None if st is None else _ptr(st), _ptr(out),
                                   C.byref(it), nthreads))
    return out, it.value


def pagerank_ref(rm: RefMatrix, degrees, alpha=0.15, iterations=10, l1_tolerance=None, dangling="uniform",
                 start=None):
    """cmv::pagerank with RefKernel(compress(A^T)) (pagerank.hpp:48-61,100-102)."""
    deg = np.ascontiguousarray(degrees, dtype=np.uint32)
    out = np.empty(len(deg), dtype=np.float64)
    it = C.c_uint32()
    st = None if start is None else np.ascontiguousarray(start, dtype=np.float64)
    _chk(lib().oracle_pagerank_ref(rm.h, _ptr(deg), alpha, iterations, -1.0 if l1_tolerance is None else l1_tolerance,
                                   0 if dangling == "uniform" else 1, None if st is None else _ptr(st), _ptr(out),
                                   C.byref(it)))
    return out, it.value


# ---- biclique covers (reference include/cmv/biclique.hpp) ----
# Test infrastructure: sequential restatements used only as the checker.

def matvec_biclique(n, bicliques, residual, x):
    """cmv::matvec_biclique_into (biclique.hpp:39-46): y = 0;
    per biclique r, c_r = sum of x over C_r (in order), added to y[i] for
    every i in S_r; per residual edge (i, j), y[i] += x[j].  Returns
    (y, c, adds) with adds = compressed_size = sum |S_r| + |C_r| + |residual|."""
    x = np.asarray(x, dtype=np.float64)
    if len(x) != n:
        raise ValueError("matvec_biclique: dimension mismatch")
    y = np.zeros(n)
    cs = []
    adds = 0
    for sources, targets in bicliques:
        c = 0.0
        for j in targets:
            c += x[j]
        cs.append(c)
        for i in sources:
            y[i] += c
        adds += len(sources) + len(targets)
    for i, j in residual:
        y[i] += x[j]
        adds += 1
    return y, cs, adds


def verify_cover(n, bicliques, residual, rows):
    """cmv::verify_cover (biclique.hpp:63-64): materialise the
    cover's edge multiset and compare it with the graph's (duplicates across
    parts make it differ)."""
    if len(rows) != n:
        return False
    got = []
    for sources, targets in bicliques:
        if len(sources) == 0 or len(targets) == 0:
            return False
        got.extend((int(i), int(j)) for i in sources for j in targets)
    got.extend((int(i), int(j)) for i, j in residual)
    want = [(u, int(v)) for u in range(n) for v in rows[u]]
    return sorted(got) == sorted(want)


# ---------------------------------------------------------------------------
# workload generators (oracle/_build/libcmv_gen.so: the product's host generator
# source compiled alone), so bench.py's CPU reference arm never loads libcmvg.so
_GEN = os.path.join(_HERE, "_build", "libcmv_gen.so")
_gen = None


def gen_lib() -> C.CDLL:
    global _gen
    if _gen is None:
        if not os.path.exists(_GEN):
            build()
        L = C.CDLL(_GEN)
        for k, (r, a) in {
            "gen_copy_model": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64, C.POINTER(_P)]),
            "gen_social": (C.c_int, [C.c_uint32, C.c_uint64, C.POINTER(_P)]),
            "gen_n": (C.c_uint32, [_P]),
            "gen_m": (C.c_uint64, [_P]),
            "gen_row_offsets": (_P, [_P]),
            "gen_cols": (_P, [_P]),
            "gen_free": (None, [_P]),
        }.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _gen = L
    return _gen


def _gen_arrays(h):
    L = gen_lib()
    try:
        n, m = int(L.gen_n(h)), int(L.gen_m(h))
        ro = _view(L.gen_row_offsets(h), n + 1, np.uint64).copy()
        co = _view(L.gen_cols(h), m, np.uint32).copy()
    finally:
        L.gen_free(h)
    return n, ro, co


def generate_copy_model(n, mean_degree, p_ref=0.7, p_copy=0.8, seed=0x170807271):
    """(n, row_offsets u64[n+1], columns u32[m]) of the seeded copy model."""
    h = _P()
    if gen_lib().gen_copy_model(n, mean_degree, p_ref, p_copy, seed, C.byref(h)):
        raise RuntimeError("gen_copy_model failed")
    return _gen_arrays(h)


def generate_social(n, seed=0x170807271 + 4):
    h = _P()
    if gen_lib().gen_social(n, seed, C.byref(h)):
        raise RuntimeError("gen_social failed")
    return _gen_arrays(h)
