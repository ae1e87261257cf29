"""B200-native compressed adjacency-matrix products (arXiv:1708.07271).

Python mirror of the reference's C++ operator surface (reference
``proj/include/cmv/*.hpp``), calling the sm_100a kernels through the C ABI in
``include/cmvg.h`` (``libcmvg.so``, built in-tree).  There is no CPU fallback:
every product runs on the GPU, and importing a handle without the built
library raises.

Reference name            -> here
``cmv::CsrGraph``         -> :class:`CsrGraph` (host)
``cmv::compress``         -> :meth:`BvStream.encode` (BV stream instead of A')
``cmv::reconstruct_graph``-> :meth:`BvGraph.decode_csr` (device)
``cmv::matvec_ref[_into]``-> :meth:`BvGraph.matvec` (form ``"gather"``)
``cmv::matvec_ref_left``  -> :meth:`BvGraph.matvec` (form ``"scatter"``)
``cmv::MatvecKernel``     -> :class:`MatvecKernel`, :class:`BvGpuKernel`
``cmv::pagerank``         -> :func:`pagerank`
``cmv::stats``            -> :meth:`BvGraph.info`, :meth:`BvStream.stats`
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
import warnings
from typing import Optional

import numpy as np

__all__ = [
    "CmvgError", "FormatError", "CorruptionError", "UnsupportedError",
    "CsrGraph", "BvParams", "BvStream", "BvGraph", "CreateOptions", "BicliqueCover", "BicliqueKernel",
    "MatvecKernel", "BvGpuKernel", "DanglingPolicy", "PageRankConfig", "PageRankResult",
    "pagerank", "library_path", "load_library", "CompressionStats", "compression_stats", "PageRankEquivalence",
    "pagerank_equivalence_check",
]

_HERE = os.path.dirname(os.path.abspath(__file__))


def library_path() -> str:
    """The in-tree libcmvg.so (CMVG_LIBRARY overrides it: A/B builds of the same sources)."""
    return os.environ.get("CMVG_LIBRARY") or os.path.join(_HERE, "libcmvg.so")


# ---------------------------------------------------------------------------
# errors (cmvg.h status codes -> the reference's exception types)
class CmvgError(RuntimeError):
    pass


class FormatError(CmvgError):  # cmv::FormatError (rmv_io.hpp:13-16)
    pass


class CorruptionError(CmvgError):  # cmv::CorruptionError (rmv_io.hpp:19-22)
    pass


class UnsupportedError(CmvgError):
    pass


_OK, _INVALID, _RANGE, _FORMAT, _CORRUPT, _CUDA, _NOMEM, _UNSUP = 0, 1, 2, 3, 4, 5, 6, 7


class _BvParamsC(C.Structure):
    _fields_ = [("window", C.c_uint32), ("max_ref", C.c_uint32), ("min_interval", C.c_uint32),
                ("zeta_k", C.c_uint32), ("segment_rows", C.c_uint32)]


class _BvStatsC(C.Structure):
    _fields_ = [("stream_bits", C.c_uint64), ("rows_with_ref", C.c_uint64), ("copied_edges", C.c_uint64),
                ("interval_edges", C.c_uint64), ("intervals", C.c_uint64), ("residual_edges", C.c_uint64),
                ("minus_edges", C.c_uint64), ("max_depth", C.c_uint32), ("nsegments", C.c_uint32)]


class _OptsC(C.Structure):
    _fields_ = [("device", C.c_int), ("block_rows", C.c_uint32), ("lanes", C.c_uint32), ("window", C.c_uint32),
                ("stream_cap_words", C.c_uint32), ("interval_mode", C.c_uint32), ("row_begin", C.c_uint32),
                ("row_end", C.c_uint32)]


class _InfoC(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("row_begin", C.c_uint32), ("row_end", C.c_uint32),
                ("bv_stream_bits", C.c_uint64), ("bvd_row_bits", C.c_uint64), ("bvd_stream_bytes", C.c_uint64),
                ("bvd_lane_table_bytes", C.c_uint64), ("bvd_block_table_bytes", C.c_uint64),
                ("block_rows", C.c_uint32), ("lanes", C.c_uint32), ("window", C.c_uint32), ("nblocks", C.c_uint32),
                ("max_depth", C.c_uint32), ("interval_mode", C.c_uint32), ("adds_per_product", C.c_uint64),
                ("device_bytes", C.c_uint64), ("bvd_codes", C.c_uint64), ("max_block_words", C.c_uint32),
                ("stream_cap_words", C.c_uint32), ("window_coverage", C.c_double),
                ("bvs_stream_bytes", C.c_uint64), ("bvs_max_block_words", C.c_uint32),
                ("bvs_stream_cap_words", C.c_uint32), ("bvs_p995_block_words", C.c_uint32), ("bvs_pad", C.c_uint32),
                ("bvs_slices", C.c_uint64), ("bvs_heavy_rows", C.c_uint64), ("bvs_lane_words", C.c_uint64),
                ("bvs_lane_words_used", C.c_uint64), ("bvs_lane_iters", C.c_uint64),
                ("bvs_lane_iters_used", C.c_uint64), ("bvt_stream_bytes", C.c_uint64), ("bvt_entries", C.c_uint64),
                ("bvt_far_slots", C.c_uint64), ("bvt_heavy_targets", C.c_uint64), ("bvt_slices", C.c_uint64),
                ("bvf_stream_bytes", C.c_uint64), ("bvf_terms", C.c_uint64), ("bvf_pad_terms", C.c_uint64),
                ("bvf_slot_terms", C.c_uint64), ("bvf_esc_terms", C.c_uint64), ("bvf_esc_blocks", C.c_uint64),
                ("bvf_max_K", C.c_uint32), ("bvf_min_cbits", C.c_uint32)]


_lib_handle: Optional[C.CDLL] = None

# (name, restype, argtypes)
_P = C.c_void_p
_SIGS = [
    ("cmvg_last_error", C.c_char_p, []),
    ("cmvg_csr_from_arrays", C.c_int, [C.c_uint32, _P, _P, C.POINTER(_P)]),
    ("cmvg_gen_copy_model", C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64, C.POINTER(_P)]),
    ("cmvg_gen_social", C.c_int, [C.c_uint32, C.c_uint64, C.POINTER(_P)]),
    ("cmvg_csr_transpose", C.c_int, [_P, C.POINTER(_P)]),
    ("cmvg_csr_n", C.c_uint32, [_P]),
    ("cmvg_csr_m", C.c_uint64, [_P]),
    ("cmvg_csr_row_offsets", _P, [_P]),
    ("cmvg_csr_cols", _P, [_P]),
    ("cmvg_csr_free", None, [_P]),
    ("cmvg_bv_encode", C.c_int, [_P, C.POINTER(_BvParamsC), C.POINTER(_P)]),
    ("cmvg_bv_from_words", C.c_int, [C.c_uint32, C.c_uint64, C.POINTER(_BvParamsC), _P, C.c_uint64, _P,
                                     C.POINTER(_P)]),
    ("cmvg_bv_decode_host", C.c_int, [_P, C.POINTER(_P)]),
    ("cmvg_bv_reconstruct_row", C.c_int, [_P, C.c_uint32, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    ("cmvg_bv_get_stats", C.c_int, [_P, C.POINTER(_BvStatsC)]),
    ("cmvg_bv_words", _P, [_P, C.POINTER(C.c_uint64)]),
    ("cmvg_bv_segment_offsets", _P, [_P, C.POINTER(C.c_uint64)]),
    ("cmvg_bv_free", None, [_P]),
    ("cmvg_default_opts", None, [C.POINTER(_OptsC)]),
    ("cmvg_create", C.c_int, [_P, C.POINTER(_OptsC), C.POINTER(_P)]),
    ("cmvg_destroy", C.c_int, [_P]),
    ("cmvg_layout_info", C.c_int, [_P, C.POINTER(_OptsC), C.POINTER(_InfoC)]),
    ("cmvg_layout_export", C.c_int, [_P, C.POINTER(_OptsC), C.POINTER(_P)]),
    ("cmvg_bvf_export", C.c_int, [_P, _P, C.c_uint64, _P, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                                  C.POINTER(C.c_int)]),
    ("cmvg_layout_words", _P, [_P, C.POINTER(C.c_uint64)]),
    ("cmvg_layout_blocks", _P, [_P, C.POINTER(C.c_uint32)]),
    ("cmvg_layout_swords", _P, [_P, C.POINTER(C.c_uint64)]),
    ("cmvg_layout_sblocks", _P, [_P, C.POINTER(C.c_uint32)]),
    ("cmvg_layout_twords", _P, [_P, C.POINTER(C.c_uint64)]),
    ("cmvg_layout_tblocks", _P, [_P, C.POINTER(C.c_uint32)]),
    ("cmvg_layout_fwords", _P, [_P, C.POINTER(C.c_uint64)]),
    ("cmvg_layout_fblocks", _P, [_P, C.POINTER(C.c_uint32)]),
    ("cmvg_layout_free", None, [_P]),
    ("cmvg_graph_info_get", C.c_int, [_P, C.POINTER(_InfoC)]),
    ("cmvg_dimension", C.c_uint32, [_P]),
    ("cmvg_adds_per_product", C.c_uint64, [_P]),
    ("cmvg_matvec_f64", C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P]),
    ("cmvg_matvec_f32", C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P]),
    ("cmvg_matmat_f32", C.c_int, [_P, _P, _P, C.c_uint32, C.c_int, _P]),
    ("cmvg_decode_csr", C.c_int, [_P, _P, _P, C.c_int, _P]),
    ("cmvg_pagerank", C.c_int, [_P, _P, C.c_double, C.c_uint32, C.c_double, C.c_int, _P, C.POINTER(C.c_uint32),
                                C.c_int, _P]),
    ("cmvg_read_set", C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    ("cmvg_pagerank_ex", C.c_int, [_P, _P, C.c_double, C.c_uint32, C.c_double, C.c_int, _P, _P,
                                   C.POINTER(C.c_uint32), C.c_int, _P]),
    ("cmvg_pagerank_step_push", C.c_int, [_P, _P, _P, C.c_double, C.c_double, C.c_int, _P, _P, _P, _P, _P, _P, _P]),
    ("cmvg_pagerank_step", C.c_int, [_P, _P, _P, C.c_double, C.c_double, C.c_int, _P, _P, _P, _P, _P]),
    ("cmvg_pagerank_step_dev", C.c_int, [_P, _P, _P, C.c_double, _P, C.c_int, _P, _P, _P, _P, _P, _P, _P]),
    ("cmvg_csr_matvec_f64", C.c_int, [C.c_uint32, C.c_uint64, _P, _P, _P, _P, _P]),
    ("cmvg_bv_save", C.c_int, [_P, C.c_char_p]),
    ("cmvg_bv_load", C.c_int, [C.c_char_p, C.POINTER(_P)]),
    ("cmvg_bv_serialize", C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    ("cmvg_bv_deserialize", C.c_int, [_P, C.c_uint64, C.POINTER(_P)]),
    ("cmvg_bv_describe", C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(_BvParamsC)]),
    ("cmvg_bicover_extract", C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(_P)]),
    ("cmvg_bicover_from_arrays", C.c_int, [C.c_uint32, C.c_uint64, _P, _P, _P, _P, C.c_uint64, _P, C.POINTER(_P)]),
    ("cmvg_bicover_sizes", C.c_int, [_P] + [C.POINTER(C.c_uint32)] + [C.POINTER(C.c_uint64)] * 5),
    ("cmvg_bicover_export", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("cmvg_bicover_verify", C.c_int, [_P, _P, C.POINTER(C.c_int)]),
    ("cmvg_bicover_save", C.c_int, [_P, C.c_char_p]),
    ("cmvg_bicover_load", C.c_int, [C.c_char_p, C.POINTER(_P)]),
    ("cmvg_bicover_matvec_f64", C.c_int, [_P, _P, _P, C.c_int, _P]),
    ("cmvg_bicover_free", None, [_P]),
]

EXPORTED_SYMBOLS = [s[0] for s in _SIGS]


def load_library() -> C.CDLL:
    """Load libcmvg.so (in-tree).  Raises if it has not been built: there is
    deliberately no fallback implementation."""
    global _lib_handle
    if _lib_handle is None:
        path = library_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(path)
        for name, res, args in _SIGS:
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib_handle = lib
    return _lib_handle


def _check(rc: int) -> None:
    if rc == _OK:
        return
    msg = load_library().cmvg_last_error().decode(errors="replace")
    if rc == _INVALID:
        raise ValueError(msg)
    if rc == _RANGE:
        raise IndexError(msg)
    if rc == _FORMAT:
        raise FormatError(msg)
    if rc == _CORRUPT:
        raise CorruptionError(msg)
    if rc == _UNSUP:
        raise UnsupportedError(msg)
    if rc == _NOMEM:
        raise MemoryError(msg)
    raise CmvgError(f"cmvg error {rc}: {msg}")


def _np_view(ptr: int, count: int, dtype) -> np.ndarray:
    if count == 0:
        return np.zeros(0, dtype=dtype)
    itemsize = np.dtype(dtype).itemsize
    buf = (C.c_char * (count * itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count)


# ---------------------------------------------------------------------------
class CsrGraph:
    """Host CSR adjacency (cmv::CsrGraph, csr.hpp:16-36) owned by the library."""

    def __init__(self, handle: int):
        self._h = _P(handle)
        lib = load_library()
        self.n = int(lib.cmvg_csr_n(self._h))
        self.m = int(lib.cmvg_csr_m(self._h))

    @classmethod
    def from_arrays(cls, n: int, row_offsets, columns) -> "CsrGraph":
        ro = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        co = np.ascontiguousarray(columns, dtype=np.uint32)
        if ro.shape != (n + 1,):
            raise ValueError("row_offsets must have n+1 entries")
        out = _P()
        _check(load_library().cmvg_csr_from_arrays(n, ro.ctypes.data, co.ctypes.data if co.size else None,
                                                   C.byref(out)))
        return cls(out.value)

    @classmethod
    def copy_model(cls, n: int, mean_degree: float, p_ref: float = 0.7, p_copy: float = 0.8,
                   seed: int = 0x170807271) -> "CsrGraph":
        out = _P()
        _check(load_library().cmvg_gen_copy_model(n, mean_degree, p_ref, p_copy, seed, C.byref(out)))
        return cls(out.value)

    @classmethod
    def social(cls, n: int, seed: int = 0x170807271 + 4) -> "CsrGraph":
        out = _P()
        _check(load_library().cmvg_gen_social(n, seed, C.byref(out)))
        return cls(out.value)

    def transpose(self) -> "CsrGraph":
        out = _P()
        _check(load_library().cmvg_csr_transpose(self._h, C.byref(out)))
        return CsrGraph(out.value)

    @property
    def row_offsets(self) -> np.ndarray:
        return _np_view(load_library().cmvg_csr_row_offsets(self._h), self.n + 1, np.uint64)

    @property
    def columns(self) -> np.ndarray:
        return _np_view(load_library().cmvg_csr_cols(self._h) or 0, self.m, np.uint32)

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets).astype(np.uint32)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib_handle is not None:
            _lib_handle.cmvg_csr_free(h)
            self._h = None


@dataclasses.dataclass
class BvParams:
    """BV encoding parameters (BASELINE.json configs: w=7, R=3 / unbounded, Lmin=4, zeta_3)."""
    window: int = 7
    max_ref: int = 3  # 0 = unbounded chains
    min_interval: int = 4
    zeta_k: int = 3
    segment_rows: int = 1024

    def _c(self) -> _BvParamsC:
        return _BvParamsC(self.window, self.max_ref, self.min_interval, self.zeta_k, self.segment_rows)


class BvStream:
    """Canonical Boldi-Vigna stream (host).  ``stats()['stream_bits']`` is S."""

    def __init__(self, handle: int, n: int, m: int, params: BvParams):
        self._h = _P(handle)
        self.n, self.m, self.params = n, m, params

    @classmethod
    def encode(cls, g: CsrGraph, params: Optional[BvParams] = None) -> "BvStream":
        params = params or BvParams()
        out = _P()
        pc = params._c()
        _check(load_library().cmvg_bv_encode(g._h, C.byref(pc), C.byref(out)))
        return cls(out.value, g.n, g.m, params)

    @classmethod
    def from_words(cls, n: int, m: int, params: BvParams, words: np.ndarray, nbits: int,
                   segment_offsets: np.ndarray) -> "BvStream":
        w = np.ascontiguousarray(words, dtype=np.uint32)
        s = np.ascontiguousarray(segment_offsets, dtype=np.uint64)
        out = _P()
        pc = params._c()
        _check(load_library().cmvg_bv_from_words(n, m, C.byref(pc), w.ctypes.data if w.size else None, nbits,
                                                 s.ctypes.data, C.byref(out)))
        return cls(out.value, n, m, params)

    # ---- CBV1 container (the reference's RMV1 model: save_rmv / load_rmv /
    # encode_rmv / decode_rmv, rmv_io.hpp:31-49) ----
    @classmethod
    def _adopt(cls, handle: int) -> "BvStream":
        n, m, pc = C.c_uint32(), C.c_uint64(), _BvParamsC()
        lib = load_library()
        rc = lib.cmvg_bv_describe(_P(handle), C.byref(n), C.byref(m), C.byref(pc))
        if rc:
            lib.cmvg_bv_free(_P(handle))
            _check(rc)
        return cls(handle, n.value, m.value, BvParams(pc.window, pc.max_ref, pc.min_interval, pc.zeta_k,
                                                      pc.segment_rows))

    def save(self, path: str) -> None:
        """Write the stream as a CBV1 container (deterministic bytes)."""
        _check(load_library().cmvg_bv_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str) -> "BvStream":
        """Read a CBV1 container; FormatError (bad magic / version) or
        CorruptionError (truncation, trailing bytes, checksum, invariants)."""
        out = _P()
        _check(load_library().cmvg_bv_load(os.fsencode(path), C.byref(out)))
        return cls._adopt(out.value)

    def to_bytes(self) -> bytes:
        size = C.c_uint64()
        lib = load_library()
        _check(lib.cmvg_bv_serialize(self._h, None, 0, C.byref(size)))
        buf = (C.c_uint8 * size.value)()
        _check(lib.cmvg_bv_serialize(self._h, buf, size.value, C.byref(size)))
        return bytes(buf)

    @classmethod
    def from_bytes(cls, data: bytes) -> "BvStream":
        out = _P()
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data) if data else None
        _check(load_library().cmvg_bv_deserialize(buf, len(data), C.byref(out)))
        return cls._adopt(out.value)

    def stats(self) -> dict:
        st = _BvStatsC()
        _check(load_library().cmvg_bv_get_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in _BvStatsC._fields_}

    def words(self) -> np.ndarray:
        nw = C.c_uint64()
        p = load_library().cmvg_bv_words(self._h, C.byref(nw))
        return _np_view(p or 0, nw.value, np.uint32).copy()

    def segment_offsets(self) -> np.ndarray:
        cnt = C.c_uint64()
        p = load_library().cmvg_bv_segment_offsets(self._h, C.byref(cnt))
        return _np_view(p, cnt.value, np.uint64).copy()

    def layout_info(self, options: Optional["CreateOptions"] = None) -> dict:
        """Sizes of the device layout for `options`, built on the host (no GPU)."""
        oc = (options or CreateOptions())._c()
        inf = _InfoC()
        _check(load_library().cmvg_layout_info(self._h, C.byref(oc), C.byref(inf)))
        return {f: getattr(inf, f) for f, _ in _InfoC._fields_}

    def layout_export(self, options: Optional["CreateOptions"] = None, sliced: bool = False, kind: str = ""):
        """(words u32[], blocks u32[nblocks, 8]) of a device layout built on the
        host: BV-D (default), BV-S (sliced=True or kind="bvs"), BV-F
        (kind="bvf") or BV-T (kind="bvt")."""
        kind = kind or ("bvs" if sliced else "bvd")
        oc = (options or CreateOptions())._c()
        h = _P()
        lib = load_library()
        _check(lib.cmvg_layout_export(self._h, C.byref(oc), C.byref(h)))
        try:
            nw, nb = C.c_uint64(), C.c_uint32()
            fw, fb = {"bvd": (lib.cmvg_layout_words, lib.cmvg_layout_blocks),
                      "bvs": (lib.cmvg_layout_swords, lib.cmvg_layout_sblocks),
                      "bvf": (lib.cmvg_layout_fwords, lib.cmvg_layout_fblocks),
                      "bvt": (lib.cmvg_layout_twords, lib.cmvg_layout_tblocks)}[kind]
            w = _np_view(fw(h, C.byref(nw)), nw.value, np.uint32).copy()
            b = _np_view(fb(h, C.byref(nb)), nb.value * 8, np.uint32).reshape(-1, 8).copy()
        finally:
            lib.cmvg_layout_free(h)
        return w, b

    def reconstruct_row(self, i: int) -> np.ndarray:
        """cmv::reconstruct_row (ref_matrix.hpp:71-73): row i of the source
        adjacency, decoded from its segment of the stream; IndexError (the
        reference's std::out_of_range) if i >= n."""
        lib = load_library()
        if i < 0:
            raise IndexError("reconstruct_row: row index out of range")
        if i >= self.n:
            raise IndexError("reconstruct_row: row index out of range")
        d = C.c_uint64()
        _check(lib.cmvg_bv_reconstruct_row(self._h, i, None, 0, C.byref(d)))
        out = np.empty(d.value, dtype=np.uint32)
        _check(lib.cmvg_bv_reconstruct_row(self._h, i, out.ctypes.data, d.value, C.byref(d)))
        return out

    def decode_host(self) -> CsrGraph:
        """CPU decode (the handle builder's path); tests compare it with the GPU decoder."""
        out = _P()
        _check(load_library().cmvg_bv_decode_host(self._h, C.byref(out)))
        return CsrGraph(out.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib_handle is not None:
            _lib_handle.cmvg_bv_free(h)
            self._h = None


@dataclasses.dataclass
class CreateOptions:
    device: int = 0
    block_rows: int = 1024
    lanes: int = 256
    window: int = 1536
    stream_cap_words: int = 0  # 0 = auto (covers 99.5% of blocks)
    interval_mode: str = "prefix"  # or "direct"
    row_begin: int = 0
    row_end: int = 0  # 0 = n

    def _c(self) -> _OptsC:
        mode = {"prefix": 0, "direct": 1}[self.interval_mode]
        return _OptsC(self.device, self.block_rows, self.lanes, self.window, self.stream_cap_words, mode,
                      self.row_begin, self.row_end)


def _is_torch(t) -> bool:
    return type(t).__module__.startswith("torch")


def _ptr_and_kind(t, dtype):
    """(pointer, ptr_kind) for a numpy array (HOST) or a CUDA torch tensor (DEVICE)."""
    if _is_torch(t):
        import torch
        want = {np.float64: torch.float64, np.float32: torch.float32, np.uint32: torch.int32,
                np.uint64: torch.int64}[dtype]
        if t.dtype != want and not (dtype in (np.uint32, np.uint64) and t.dtype in (torch.int32, torch.int64)):
            raise TypeError(f"expected {want}, got {t.dtype}")
        if not t.is_cuda:
            raise ValueError("torch tensors must live on the GPU; pass numpy arrays for host buffers")
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return t.data_ptr(), 1
    if not isinstance(t, np.ndarray) or t.dtype != dtype or not t.flags.c_contiguous:
        raise TypeError(f"expected a C-contiguous numpy array of {np.dtype(dtype)}")
    return t.ctypes.data, 0


def _stream_of(*ts) -> Optional[int]:
    for t in ts:
        if _is_torch(t) and t.is_cuda:
            import torch
            return torch.cuda.current_stream(t.device).cuda_stream
    return None


def csr_matvec_device(row_offsets, cols, x, y=None, stream: Optional[int] = None):
    """Uncompressed y = A x^T on the GPU (the reference's matvec_csr,
    csr.hpp:48-55) from CUDA tensors: row_offsets int64[n+1], cols int32[m],
    x float64[n].  The comparison point for the compressed product at equal
    hardware."""
    import torch
    for t in (row_offsets, cols, x):
        if not (_is_torch(t) and t.is_cuda and t.is_contiguous()):
            raise ValueError("csr_matvec_device takes contiguous CUDA tensors")
    if row_offsets.dtype != torch.int64 or cols.dtype != torch.int32 or x.dtype != torch.float64:
        raise TypeError("expected int64 row offsets, int32 columns, float64 x")
    n = row_offsets.numel() - 1
    if x.numel() != n:
        raise ValueError(f"x has {x.numel()} entries, the matrix {n} columns")
    if y is None:
        y = torch.empty(n, dtype=torch.float64, device=x.device)
    st = stream if stream is not None else _stream_of(x)
    _check(load_library().cmvg_csr_matvec_f64(n, cols.numel(), row_offsets.data_ptr(), cols.data_ptr(),
                                              x.data_ptr(), y.data_ptr(), st))
    return y


UNBOUNDED_ROUNDS = (1 << 64) - 1  # cmv::kUnboundedRounds (biclique.hpp:46-47)


class BicliqueCover:
    """Edge-disjoint biclique cover of a graph plus residual edges (the
    reference's cmv::BicliqueCover, biclique.hpp:24-38) with its GPU product.
    ``compressed_size`` = sum |S_r| + |C_r| + |residual|, the adds of one
    product (biclique.hpp:33-34)."""

    def __init__(self, handle: int):
        self._h = _P(handle)
        self._sz = None  # the cover is immutable: sizes cached on first use

    @classmethod
    def extract_greedy(cls, g: CsrGraph, min_gain: int = 1, max_rounds: int = UNBOUNDED_ROUNDS,
                       per_round: int = 1) -> "BicliqueCover":
        """cmv::extract_greedy (biclique.hpp:58-61).  per_round=1 emits the
        best candidate per round (the reference's rule); 0 emits every
        still-valid candidate of a round in gain order (large graphs)."""
        out = _P()
        _check(load_library().cmvg_bicover_extract(g._h, min_gain, max_rounds, per_round, C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_lists(cls, n: int, bicliques, residual) -> "BicliqueCover":
        """From [(sources, targets), ...] and [(u, v), ...] (ids ascending)."""
        src = [np.asarray(s, dtype=np.uint32) for s, _ in bicliques]
        tgt = [np.asarray(t, dtype=np.uint32) for _, t in bicliques]
        so = np.zeros(len(src) + 1, dtype=np.uint64)
        to = np.zeros(len(tgt) + 1, dtype=np.uint64)
        so[1:] = np.cumsum([len(a) for a in src]) if src else []
        to[1:] = np.cumsum([len(a) for a in tgt]) if tgt else []
        sa = np.concatenate(src) if src else np.zeros(1, dtype=np.uint32)
        ta = np.concatenate(tgt) if tgt else np.zeros(1, dtype=np.uint32)
        res = np.ascontiguousarray(np.asarray(residual, dtype=np.uint32).reshape(-1, 2))
        out = _P()
        _check(load_library().cmvg_bicover_from_arrays(
            n, len(src), so.ctypes.data, sa.ctypes.data, to.ctypes.data, ta.ctypes.data, len(res),
            res.ctypes.data if len(res) else None, C.byref(out)))
        return cls(out.value)

    def _sizes(self):
        if self._sz is None:
            n, v = C.c_uint32(), [C.c_uint64() for _ in range(5)]
            _check(load_library().cmvg_bicover_sizes(self._h, C.byref(n), *[C.byref(a) for a in v]))
            self._sz = (n.value,) + tuple(a.value for a in v)
        return self._sz

    @property
    def n(self) -> int:
        return self._sizes()[0]

    @property
    def compressed_size(self) -> int:
        return self._sizes()[5]

    def lists(self):
        """([(sources, targets), ...], residual (k, 2) uint32)."""
        n, nb, ns, nt, nr, _ = self._sizes()
        so, to = np.zeros(nb + 1, dtype=np.uint64), np.zeros(nb + 1, dtype=np.uint64)
        sa, ta = np.zeros(max(ns, 1), dtype=np.uint32), np.zeros(max(nt, 1), dtype=np.uint32)
        res = np.zeros((max(nr, 1), 2), dtype=np.uint32)
        _check(load_library().cmvg_bicover_export(self._h, so.ctypes.data, sa.ctypes.data, to.ctypes.data,
                                                  ta.ctypes.data, res.ctypes.data))
        bl = [(sa[so[r]:so[r + 1]].copy(), ta[to[r]:to[r + 1]].copy()) for r in range(nb)]
        return bl, res[:nr].copy()

    def verify(self, g: CsrGraph) -> bool:
        """cmv::verify_cover (biclique.hpp:63-64)."""
        ok = C.c_int()
        _check(load_library().cmvg_bicover_verify(self._h, g._h, C.byref(ok)))
        return bool(ok.value)

    def save(self, path: str) -> None:
        _check(load_library().cmvg_bicover_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str) -> "BicliqueCover":
        out = _P()
        _check(load_library().cmvg_bicover_load(os.fsencode(path), C.byref(out)))
        return cls(out.value)

    def matvec(self, x, y=None, stream: Optional[int] = None):
        """y = A x on the GPU (cmv::matvec_biclique_into, biclique.hpp:39-46):
        numpy in/out (HOST) or CUDA torch tensors (DEVICE)."""
        n = self.n
        if len(x) != n:
            raise ValueError(f"x has {len(x)} entries, the cover {n} vertices")
        if y is None:
            if _is_torch(x):
                import torch
                y = torch.empty(n, dtype=torch.float64, device=x.device)
            else:
                y = np.empty(n, dtype=np.float64)
        xp, kind = _ptr_and_kind(x, np.float64)
        yp, kind2 = _ptr_and_kind(y, np.float64)
        if kind != kind2:
            raise ValueError("x and y must both be host arrays or both CUDA tensors")
        st = stream if stream is not None else _stream_of(x, y)
        _check(load_library().cmvg_bicover_matvec_f64(self._h, xp, yp, kind, st))
        return y

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib_handle is not None:
            _lib_handle.cmvg_bicover_free(h)
            self._h = None


class BicliqueKernel:
    """MatvecKernel over a biclique cover of A^T (for pagerank)."""

    def __init__(self, cover_of_transpose: BicliqueCover):
        self.cover = cover_of_transpose

    def dimension(self) -> int:
        return self.cover.n

    def multiply(self, x, y) -> None:
        self.cover.matvec(x, y)

    def adds_per_product(self) -> int:
        return self.cover.compressed_size


class BvGraph:
    """Device handle over a BV stream (one GPU; optionally one row shard)."""

    def __init__(self, stream: BvStream, options: Optional[CreateOptions] = None):
        self.options = options or CreateOptions()
        out = _P()
        oc = self.options._c()
        _check(load_library().cmvg_create(stream._h, C.byref(oc), C.byref(out)))
        self._h = out
        self.n = stream.n
        self.m = stream.m
        info = self.info()
        self.row_begin, self.row_end = info["row_begin"], info["row_end"]

    def info(self) -> dict:
        inf = _InfoC()
        _check(load_library().cmvg_graph_info_get(self._h, C.byref(inf)))
        return {f: getattr(inf, f) for f, _ in _InfoC._fields_}

    def dimension(self) -> int:
        return int(load_library().cmvg_dimension(self._h))

    def adds_per_product(self) -> int:
        return int(load_library().cmvg_adds_per_product(self._h))

    def matvec(self, x, y=None, form: str = "gather", stream: Optional[int] = None):
        """y = A x^T ("gather") or y = x A: "scatter" on A's own compression
        (atomic-free segmented sums), or "left" as (A^T) x on the transpose's
        compression -- the reference's matvec_ref_left, built on the GPU on
        first use (whole-graph handles).  numpy in -> numpy out (host copies
        inside the call); CUDA tensors in -> CUDA tensors out."""
        formc = {"gather": 0, "scatter": 1, "left": 2}[form]
        dtype = np.float64 if (x.dtype == np.float64 or str(x.dtype) == "torch.float64") else np.float32
        nout = (self.row_end - self.row_begin) if form == "gather" else self.n
        if len(x) != self.n:
            raise ValueError(f"dimension mismatch: x has {len(x)} entries, graph has {self.n}")
        if y is None:
            if _is_torch(x):
                import torch
                y = torch.empty(nout, dtype=x.dtype, device=x.device)
            else:
                y = np.empty(nout, dtype=dtype)
        if len(y) != nout:
            raise ValueError("dimension mismatch on y")
        px, kx = _ptr_and_kind(x, dtype)
        py, ky = _ptr_and_kind(y, dtype)
        if kx != ky:
            raise ValueError("x and y must both be host arrays or both device tensors")
        st = stream if stream is not None else _stream_of(x, y)
        f = load_library().cmvg_matvec_f64 if dtype == np.float64 else load_library().cmvg_matvec_f32
        _check(f(self._h, px, py, formc, kx, st))
        return y

    def matmat(self, X, Y=None, stream: Optional[int] = None):
        """Y = A X for X of shape (n, k), float32, row-major."""
        k = X.shape[1]
        nout = self.row_end - self.row_begin
        if X.shape[0] != self.n:
            raise ValueError("dimension mismatch")
        if Y is None:
            if _is_torch(X):
                import torch
                Y = torch.empty((nout, k), dtype=X.dtype, device=X.device)
            else:
                Y = np.empty((nout, k), dtype=np.float32)
        px, kx = _ptr_and_kind(X, np.float32)
        py, ky = _ptr_and_kind(Y, np.float32)
        st = stream if stream is not None else _stream_of(X, Y)
        _check(load_library().cmvg_matmat_f32(self._h, px, py, k, kx, st))
        return Y

    def decode_csr(self):
        """Decode the canonical BV stream on the GPU (bit-exact adjacency)."""
        ro = np.empty(self.n + 1, dtype=np.uint64)
        co = np.empty(max(self.m, 1), dtype=np.uint32)
        _check(load_library().cmvg_decode_csr(self._h, ro.ctypes.data, co.ctypes.data, 0, None))
        return ro, co[: self.m]

    def decode_csr_device(self, row_offsets, cols, stream: Optional[int] = None):
        pr, _ = _ptr_and_kind(row_offsets, np.uint64)
        pc, _ = _ptr_and_kind(cols, np.uint32)
        st = stream if stream is not None else _stream_of(row_offsets)
        _check(load_library().cmvg_decode_csr(self._h, pr, pc, 1, st))

    def pagerank(self, degrees, alpha: float = 0.15, iterations: int = 10, l1_tolerance: Optional[float] = None,
                 dangling: str = "uniform", ranks=None, stream: Optional[int] = None, start=None):
        """Device-resident PageRank on a handle holding A^T; returns (ranks, iterations_run).
        `start` (a probability vector, host array or device tensor like
        `degrees`) is the starting and restart distribution (cmvg_pagerank_ex)."""
        if len(degrees) != self.n:
            raise ValueError("degree vector dimension mismatch")
        if ranks is None:
            if _is_torch(degrees):
                import torch
                ranks = torch.empty(self.n, dtype=torch.float64, device=degrees.device)
            else:
                ranks = np.empty(self.n, dtype=np.float64)
        pd, kd = _ptr_and_kind(degrees, np.uint32)
        pr, kr = _ptr_and_kind(ranks, np.float64)
        if kd != kr:
            raise ValueError("degrees and ranks must both be host arrays or both device tensors")
        it = C.c_uint32()
        st = stream if stream is not None else _stream_of(degrees, ranks)
        ps = None
        if start is not None:
            if len(start) != self.n:
                raise ValueError("pagerank: start dimension mismatch")
            if not _is_torch(start):
                start = np.ascontiguousarray(start, dtype=np.float64)
            ps, ks = _ptr_and_kind(start, np.float64)
            if ks != kd:
                raise ValueError("start must live where degrees live (host or device)")
        _check(load_library().cmvg_pagerank_ex(self._h, pd, alpha, iterations,
                                               -1.0 if l1_tolerance is None else float(l1_tolerance),
                                               {"uniform": 0, "drop": 1}[dangling], ps, pr, C.byref(it), kd, st))
        return ranks, int(it.value)

    def pagerank_step(self, q, degrees_shard, alpha, dangling_mass, dangling, p_prev, p_next, q_next, partial,
                      stream: Optional[int] = None, push_mask=None, push_dst=None):
        """One sharded PageRank iteration (device tensors); see cmvg_pagerank_step.
        With push_mask (uint8 per shard row) and push_dst (int64 device tensor
        of peer q-buffer pointers) the halo exchange is fused into the kernel
        (cmvg_pagerank_step_push)."""
        ptrs = [q.data_ptr(), degrees_shard.data_ptr(), p_prev.data_ptr() if p_prev is not None else None,
                p_next.data_ptr(), q_next.data_ptr(), partial.data_ptr()]
        st = stream if stream is not None else _stream_of(q)
        lib = load_library()
        dang = {"uniform": 0, "drop": 1}[dangling]
        if push_mask is None:
            _check(lib.cmvg_pagerank_step(self._h, ptrs[0], ptrs[1], alpha, dangling_mass, dang, ptrs[2], ptrs[3],
                                          ptrs[4], ptrs[5], st))
        else:
            _check(lib.cmvg_pagerank_step_push(self._h, ptrs[0], ptrs[1], alpha, dangling_mass, dang, ptrs[2],
                                               ptrs[3], ptrs[4], ptrs[5], push_mask.data_ptr(), push_dst.data_ptr(),
                                               st))

    def pagerank_step_dev(self, q, degrees_shard, alpha, dangling_mass, dangling, p_prev, p_next, q_next, partial,
                          stream: Optional[int] = None, push_mask=None, push_dst=None):
        """pagerank_step with the dangling mass a DEVICE tensor (its element 0;
        cmvg_pagerank_step_dev): no host synchronisation between iterations."""
        st = stream if stream is not None else _stream_of(q)
        dang = {"uniform": 0, "drop": 1}[dangling]
        _check(load_library().cmvg_pagerank_step_dev(
            self._h, q.data_ptr(), degrees_shard.data_ptr(), alpha, dangling_mass.data_ptr(), dang,
            p_prev.data_ptr() if p_prev is not None else None, p_next.data_ptr(), q_next.data_ptr(),
            partial.data_ptr(), push_mask.data_ptr() if push_mask is not None else None,
            push_dst.data_ptr() if push_dst is not None else None, st))

    def read_set(self) -> np.ndarray:
        """Sorted columns of x this handle's gather reads (x-windows + out-of-window
        columns): what a sharded PageRank must receive from the other shards."""
        lib = load_library()
        cnt = C.c_uint64()
        _check(lib.cmvg_read_set(self._h, None, 0, C.byref(cnt)))
        out = np.empty(cnt.value, dtype=np.uint32)
        _check(lib.cmvg_read_set(self._h, out.ctypes.data if cnt.value else None, cnt.value, C.byref(cnt)))
        return out

    def bvf_export(self):
        """(words u32[], blocks u32[nblocks, 8], device_built) of the BV-F layout
        this handle's products read (the same format as
        BvStream.layout_export(kind="bvf"), block offsets relative to the
        handle's first block)."""
        lib = load_library()
        nw, nb, dev = C.c_uint64(), C.c_uint32(), C.c_int()
        _check(lib.cmvg_bvf_export(self._h, None, 0, None, 0, C.byref(nw), C.byref(nb), C.byref(dev)))
        w = np.empty(nw.value, np.uint32)
        b = np.empty((nb.value, 8), np.uint32)
        _check(lib.cmvg_bvf_export(self._h, w.ctypes.data, w.size, b.ctypes.data, b.size, C.byref(nw), C.byref(nb),
                                   C.byref(dev)))
        return w, b, bool(dev.value)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib_handle is not None:
            _lib_handle.cmvg_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()


# ---------------------------------------------------------------------------
# cmv::MatvecKernel (pagerank.hpp:25-34) and the GPU drop-in
class MatvecKernel:
    """A representation of A^T able to compute y = A^T x (pagerank.hpp:25-34)."""

    def dimension(self) -> int:
        raise NotImplementedError

    def multiply(self, x, y) -> None:
        raise NotImplementedError

    def adds_per_product(self) -> int:
        raise NotImplementedError


class BvGpuKernel(MatvecKernel):
    """GPU kernel over BV(A^T): the drop-in for cmv::RefKernel (pagerank.hpp:48-61).
    ``multiply`` takes host arrays (H2D/D2H inside) or CUDA tensors."""

    def __init__(self, graph_of_transpose: BvGraph):
        self.graph = graph_of_transpose

    def dimension(self) -> int:
        return self.graph.dimension()

    def multiply(self, x, y) -> None:
        self.graph.matvec(x, y, form="gather")

    def adds_per_product(self) -> int:
        return self.graph.adds_per_product()


class DanglingPolicy(enum.Enum):  # pagerank.hpp:16
    UNIFORM = "uniform"
    DROP = "drop"


@dataclasses.dataclass
class PageRankConfig:  # pagerank.hpp:18-23
    alpha: float = 0.15
    iterations: int = 10
    l1_tolerance: Optional[float] = None
    dangling: DanglingPolicy = DanglingPolicy.UNIFORM


@dataclasses.dataclass
class PageRankResult:  # pagerank.hpp:78-81
    ranks: np.ndarray
    iterations_run: int


def pagerank(at: BvGpuKernel, degrees, cfg: Optional[PageRankConfig] = None, start=None) -> PageRankResult:
    """cmv::pagerank (pagerank.hpp:83-102) for the GPU kernel: the whole power
    iteration runs on the device.  Same validation and error behaviour
    (ValueError for the reference's std::invalid_argument)."""
    cfg = cfg or PageRankConfig()
    if not isinstance(at, BvGpuKernel):
        raise TypeError("pagerank() drives a BvGpuKernel; other kernels are out of scope here")
    if not (0.0 < cfg.alpha < 1.0):
        raise ValueError("pagerank: alpha must be in (0,1)")
    if cfg.iterations == 0:
        raise ValueError("pagerank: iterations must be > 0")
    if at.dimension() == 0:
        raise ValueError("pagerank: empty graph")
    if len(degrees) != at.dimension():
        raise ValueError("pagerank: degree vector dimension mismatch")
    deg = degrees if _is_torch(degrees) else np.ascontiguousarray(degrees, dtype=np.uint32)
    if start is not None and not _is_torch(deg):
        start = np.ascontiguousarray(start, dtype=np.float64)
    ranks, it = at.graph.pagerank(deg, cfg.alpha, cfg.iterations, cfg.l1_tolerance, cfg.dangling.value, start=start)
    return PageRankResult(ranks, it)


# ---------------------------------------------------------------------------
# cmv::stats / cmv::pagerank_equivalence_check (ref_matrix.hpp:78-89,
# pagerank.hpp:104-118)
@dataclasses.dataclass
class CompressionStats:  # ref_matrix.hpp:78-86
    n: int = 0
    m: int = 0
    m_prime: int = 0                 # entries of A' (plus + minus)
    ratio: float = 1.0               # m / m_prime
    ratio_by_convention: bool = False  # m_prime == 0
    rows_self_coded: int = 0         # rows without a reference
    max_chain: int = 0               # longest reference chain


def compression_stats(stream: "BvStream") -> CompressionStats:
    """cmv::stats for a BV stream: A' = per row the reference's skipped entries
    (minus) plus BV's extra list (intervals + residuals)."""
    st = stream.stats()
    mp = int(st["interval_edges"] + st["residual_edges"] + st["minus_edges"])
    return CompressionStats(n=stream.n, m=stream.m, m_prime=mp, ratio=(stream.m / mp) if mp else 1.0,
                            ratio_by_convention=mp == 0, rows_self_coded=int(stream.n - st["rows_with_ref"]),
                            max_chain=int(st["max_depth"]))


@dataclasses.dataclass
class PageRankEquivalence:  # pagerank.hpp:106-114
    linf: float = 0.0        # max |csr - ref| over vertices
    iterations_run: int = 0
    csr_seconds: float = 0.0
    ref_seconds: float = 0.0
    csr_adds: int = 0        # per product
    ref_adds: int = 0        # per product
    compression: CompressionStats = dataclasses.field(default_factory=CompressionStats)


def pagerank_equivalence_check(g: "CsrGraph", cfg: Optional[PageRankConfig] = None, window: int = 7,
                               device: int = 0) -> PageRankEquivalence:
    """cmv::pagerank_equivalence_check: the same PageRank with the baseline CSR
    kernel and the differential kernel, both on the GPU.  The CSR side is a
    plain sparse product of CSR(A^T) (cuSPARSE through torch, fp64) in the
    same power iteration; the differential side is this library's device
    PageRank on BV(A^T) with BV window `window`.  Timings are device time of
    the iterations."""
    import torch

    cfg = cfg or PageRankConfig()
    if window < 1:
        raise ValueError("pagerank_equivalence_check: window must be >= 1")
    dev = torch.device("cuda", device)
    at = g.transpose()
    stream = BvStream.encode(at, BvParams(window=min(window, 7)))
    dg = BvGraph(stream, CreateOptions(device=device))
    deg_np = g.out_degrees()
    deg = torch.from_numpy(deg_np.astype(np.int32)).to(dev)
    dg.pagerank(deg, cfg.alpha, 2, None, cfg.dangling.value)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p_ref, it_ref = dg.pagerank(deg, cfg.alpha, cfg.iterations, cfg.l1_tolerance, cfg.dangling.value)
    e1.record()
    torch.cuda.synchronize(dev)
    ref_s = e0.elapsed_time(e1) * 1e-3
    # baseline: CSR(A^T) y = A^T q (cuSPARSE), identical recurrence to the reference's pagerank
    n = g.n
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # torch's "sparse CSR is beta" notices
        A = torch.sparse_csr_tensor(torch.from_numpy(at.row_offsets.astype(np.int64)),
                                    torch.from_numpy(at.columns.astype(np.int64)),
                                    torch.ones(at.m, dtype=torch.float64), size=(n, n)).to(dev)
    d = deg.to(torch.float64)
    alpha = cfg.alpha
    p = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    e0.record()
    it = 0
    for it in range(1, cfg.iterations + 1):
        q = torch.where(d > 0, p / d.clamp(min=1), torch.zeros_like(p))
        dm = p[d == 0].sum() if cfg.dangling == DanglingPolicy.UNIFORM else torch.zeros((), dtype=torch.float64,
                                                                                     device=dev)
        y = torch.mv(A, q)
        nxt = alpha / n + (1.0 - alpha) * (y + dm / n)
        l1 = float((nxt - p).abs().sum()) if cfg.l1_tolerance is not None else None
        p = nxt
        if cfg.l1_tolerance is not None and l1 <= cfg.l1_tolerance:
            break
    e1.record()
    torch.cuda.synchronize(dev)
    csr_s = e0.elapsed_time(e1) * 1e-3
    return PageRankEquivalence(linf=float((p - p_ref).abs().max()), iterations_run=int(it_ref), csr_seconds=csr_s,
                               ref_seconds=ref_s, csr_adds=int(at.m), ref_adds=int(dg.adds_per_product()),
                               compression=compression_stats(stream))
